#!/bin/bash
# Full GPU suite + smoke + PCIe probe.
O=gpurun_out/r2e; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke rc=$?
timeout 120 ./build/pcie_probe > $O/pcie.log 2>&1
tail -15 $O/pytest_gpu.log; tail -2 $O/smoke.log; cat $O/pcie.log
