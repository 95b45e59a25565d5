"""ncu capture of one env-step launch -> profiles/r2/traffic_<config>_k<K>.json,
the per-launch counters bench.py attaches to its roofline line:

  python tools/traffic_r2.py <raw.csv> <details.csv> <config> <K> [note]

DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum), L2 bytes
(32 x lts__t_sectors_srcunit_tex: the SMs' L2 reads and writes), issue-slot use (average and the busiest / idlest SM
sub-partition), instructions, duration, warps per SM."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def raw_metrics(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for h, u, v in zip(hdr, units, vals):
        try:
            out[h] = (float(v.replace(",", "")), u)
        except ValueError:
            pass
    return out


def to_bytes(v, u):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return v * scale.get(u, 1)


def to_us(v, u):
    return v * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}.get(u, 1.0)


def summarize(raw_path, details_path=None):
    m = raw_metrics(raw_path)
    g = lambda k: m.get(k, (None, ""))
    dram = to_bytes(*g("dram__bytes_read.sum")) + to_bytes(*g("dram__bytes_write.sum"))
    out = dict(
        dram_bytes_per_launch=dram,
        # L2 traffic from the SMs (lts__t_bytes = 32 B sectors): reads / writes of this kernel
        lts_bytes_per_launch=32 * g("lts__t_sectors_srcunit_tex.sum")[0] if "lts__t_sectors_srcunit_tex.sum" in m else None,
        lts_read_bytes_per_launch=32 * g("lts__t_sectors_srcunit_tex_op_read.sum")[0]
        if "lts__t_sectors_srcunit_tex_op_read.sum" in m else None,
        lts_write_bytes_per_launch=32 * g("lts__t_sectors_srcunit_tex_op_write.sum")[0]
        if "lts__t_sectors_srcunit_tex_op_write.sum" in m else None,
        duration_us=to_us(*g("gpu__time_duration.sum")),
        issue_active_pct=g("smsp__issue_active.avg.pct_of_peak_sustained_active")[0],
        issue_active_pct_max_smsp=g("smsp__issue_active.max.pct_of_peak_sustained_active")[0],
        issue_active_pct_min_smsp=g("smsp__issue_active.min.pct_of_peak_sustained_active")[0],
        inst_executed=g("smsp__inst_executed.sum")[0],
        inst_executed_smsp_max=g("smsp__inst_executed.max")[0],
        inst_executed_smsp_min=g("smsp__inst_executed.min")[0],
        warps_active_per_sm=g("sm__warps_active.avg.per_cycle_active")[0],
        registers_per_thread=g("launch__registers_per_thread")[0],
        grid=g("launch__grid_size")[0],
        block=g("launch__block_size")[0],
    )
    return out


if __name__ == "__main__":
    raw, det, cfg, k = sys.argv[1:5]
    note = sys.argv[5] if len(sys.argv) > 5 else ""
    s = summarize(raw, det)
    s["source"] = f"ncu --set full --clock-control none, first timed launch of bench.py --config {cfg} --fuse {k}; {note}"
    os.makedirs(os.path.join(ROOT, "profiles", "r2"), exist_ok=True)
    dst = os.path.join(ROOT, "profiles", "r2", f"traffic_{cfg}_k{k}.json")
    json.dump(s, open(dst, "w"), indent=1)
    print(dst, json.dumps(s))
