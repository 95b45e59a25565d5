"""Turn a tools/profile_round.sh output directory into the committed
profiles/<round>/ summaries:  python tools/summarize_profiles.py gpurun_out/prof_round r1

Writes per-kernel headline metrics (details page subset), the per-launch
DRAM traffic (profiles/traffic_<config>.json, read by bench.py's roofline
`traffic`), compact launch lists with per-kernel shares, and the SASS
opcode / stall mix of the env-step kernel."""
import collections
import csv
import io
import json
import os
import sys

KEEP = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Active Warps Per Scheduler",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "Registers Per Thread", "Block Size", "Grid Size", "Dynamic Shared Memory Per Block",
        "Theoretical Occupancy", "Achieved Occupancy", "Achieved Active Warps Per SM"]
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
       "smsp__inst_executed.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__issue_active.avg.pct_of_peak_sustained_active"]


def details(path):
    rows = list(csv.reader(open(path)))
    hdr = {h: i for i, h in enumerate(rows[0])}
    out = {}
    for r in rows[1:]:
        if len(r) > hdr["Metric Name"] and r[hdr["Metric Name"]] in KEEP:
            out[r[hdr["Metric Name"]]] = f"{r[hdr['Metric Value']]} {r[hdr['Metric Unit']]}".strip()
    return out


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out, stalls = {}, {}
    for h, u, v in zip(hdr, units, vals):
        if h in RAW:
            out[h] = f"{v} {u}".strip()
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                f = float(v.replace(",", ""))
            except ValueError:
                continue
            if f >= 0.02:
                stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(f, 3)
    return out, dict(sorted(stalls.items(), key=lambda kv: -kv[1]))


def num(s):
    return float(s.split()[0].replace(",", ""))


def launches(path, top=12):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = {h: i for i, h in enumerate(rows[0])}
    per = collections.defaultdict(lambda: [0, 0.0])
    lst = []
    for r in rows[1:]:
        if len(r) <= hdr["Metric Value"] or r[hdr["Metric Name"]] != "gpu__time_duration.sum":
            continue
        k = r[hdr["Kernel Name"]]
        v = float(r[hdr["Metric Value"]].replace(",", ""))
        us = v / 1e3 if r[hdr["Metric Unit"]] == "ns" else (v if r[hdr["Metric Unit"]] == "us" else v * 1e3)
        per[k][0] += 1
        per[k][1] += us
        lst.append((r[hdr["ID"]], k[:110], round(us, 3)))
    total = sum(t for _, t in per.values()) or 1.0
    share = [(k[:110], c, round(t, 1), round(100 * t / total, 2)) for k, (c, t) in
             sorted(per.items(), key=lambda kv: -kv[1][1])[:top]]
    return lst, share, total


def sass_mix(path, top=20):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Source" in r)
    hdr = {h: i for i, h in enumerate(rows[hi])}
    ops, st = collections.Counter(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) < len(hdr):
            continue
        src = r[hdr["Source"]].strip()
        try:
            ex = int(r[hdr["Instructions Executed"]] or 0)
            smp = int(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        except (ValueError, KeyError):
            continue
        tok = src.split()
        if not tok:
            continue
        op = (tok[1] if tok[0].startswith("@") and len(tok) > 1 else tok[0]).split(".")[0]
        ops[op] += ex
        st[op] += smp
    tot, tst = sum(ops.values()) or 1, sum(st.values()) or 1
    return [(op, ex, round(100 * ex / tot, 2), round(100 * st[op] / tst, 2)) for op, ex in ops.most_common(top)]


def main(src, rnd):
    dst = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", rnd)
    os.makedirs(dst, exist_ok=True)
    summary = {}
    for f in ("env_step_psm", "env_step_ecm", "env_step_star", "policy_fwd", "mt_step_multitool", "im_step_image",
              "path_record_star"):
        d, r = os.path.join(src, f + "_details.csv"), os.path.join(src, f + "_raw.csv")
        if not os.path.exists(d):
            continue
        ent = {"details": details(d)}
        if os.path.exists(r):
            ent["raw"], ent["stalls_per_issued_instruction"] = raw(r)
            try:
                ent["dram_bytes_per_launch"] = num(ent["raw"]["dram__bytes_read.sum"]) + \
                    num(ent["raw"]["dram__bytes_write.sum"])
            except KeyError:
                pass
        s = os.path.join(src, f + "_sass.csv")
        if os.path.exists(s):
            try:
                ent["sass_opcode_mix"] = [dict(op=o, executed=e, pct_executed=p, pct_stall_samples=q)
                                          for o, e, p, q in sass_mix(s)]
            except StopIteration:
                pass
        summary[f] = ent
        if f.split("_")[0] in ("env", "mt", "im") and "dram_bytes_per_launch" in ent:
            cfg = f.split("_")[-1]
            units = {"B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            b = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                v, *u = ent["raw"][k].split()
                b += float(v.replace(",", "")) * units.get(u[0] if u else "B", 1)
            json.dump(dict(kernel=f, dram_bytes_per_launch=b, round=rnd,
                           source=f"profiles/{rnd}/ncu_summary.json (ncu --set full, one fused 250-step launch)"),
                      open(os.path.join(os.path.dirname(dst), f"traffic_{cfg}.json"), "w"), indent=1)
    for name in ("psm", "ppo"):
        p = os.path.join(src, f"launches_{name}.csv")
        if not os.path.exists(p):
            continue
        lst, share, total = launches(p)
        summary[f"launches_{name}"] = dict(total_us=round(total, 1), share=[
            dict(kernel=k, launches=c, total_us=t, pct=s) for k, c, t, s in share])
        with open(os.path.join(dst, f"launches_{name}.csv"), "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(["id", "kernel", "duration_us"])
            w.writerows(lst)
    json.dump(summary, open(os.path.join(dst, "ncu_summary.json"), "w"), indent=1)
    print(json.dumps({k: (v.get("details", {}).get("Duration"), v.get("dram_bytes_per_launch"))
                      if isinstance(v, dict) and "details" in v else v.get("total_us")
                      for k, v in summary.items()}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "r1")
