"""Summarise an ncu report (--set full) and/or a launch-list CSV into
profiles/: per kernel duration, FP64/ALU/LSU pipe utilisation, issue-slot
use, occupancy, DRAM bytes, L2 hit rate and the top stall reasons.

  python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
      --out profiles/r01_cfg2 [--pairs 4.29e9]
"""
import argparse
import csv
import io
import json
import subprocess
from collections import defaultdict

METRICS = {
    "duration_ms": "gpu__time_duration.sum",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "warp_instructions": "smsp__inst_executed.sum",
    "warps_active_per_smsp": "smsp__warps_active.avg.per_cycle_active",
    "registers": "launch__registers_per_thread",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
}
STALLS = ["math_pipe_throttle", "not_selected", "selected", "wait", "dispatch_stall", "barrier",
          "short_scoreboard", "long_scoreboard", "branch_resolving", "mio_throttle", "no_instructions"]
UNIT_SCALE = {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "s": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
              "Gbyte": 1e9}


def read_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for key, m in METRICS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                if key == "duration_ms":
                    v *= UNIT_SCALE.get(units[i], 1.0)
                if key.startswith("dram_") and units[i] in UNIT_SCALE:
                    v *= UNIT_SCALE[units[i]]
                d[key] = v
        st = {}
        for s in STALLS:
            m = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if m in hdr:
                st[s] = float(r[hdr.index(m)])
        d["stalls_per_issue"] = dict(sorted(st.items(), key=lambda kv: -kv[1])[:6])
        res.append(d)
    return res


def read_launches(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.reader(io.StringIO(txt[start:])))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", "")) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3,
                                             "nsecond": 1e-6, "msecond": 1.0}.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    return [{"kernel": k, "launches": v[0], "total_ms": v[1], "share": v[1] / tot if tot else 0}
            for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--note", default="")
    ap.add_argument("--traffic-out", help="write {dram_bytes_per_eval} here (the --set full capture "
                    "must hold exactly one evaluation's hot kernels)")
    a = ap.parse_args()
    summary = {"note": a.note}
    lines = [f"# ncu summary: {a.out}", "", a.note, ""]
    if a.launches:
        L = read_launches(a.launches)
        summary["launches"] = L
        lines += ["## Launch list (gpu__time_duration.sum, --clock-control none; cold, serialised)", "",
                  "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        lines += [f"| {x['kernel']} | {x['launches']} | {x['total_ms']:.3f} | {100 * x['share']:.1f}% |" for x in L]
        lines.append("")
    if a.rep:
        R = read_raw(a.rep)
        summary["kernels"] = R
        lines += ["## Full capture (--set full)", ""]
        for d in R:
            lines.append(f"### {d['kernel']}")
            for k in METRICS:
                if k in d:
                    lines.append(f"- {k}: {d[k]:.4g}")
            lines.append(f"- top stalls (warps per issue): {d['stalls_per_issue']}")
            lines.append("")
    json.dump(summary, open(a.out + ".json", "w"), indent=1)
    if a.traffic_out and a.rep:
        tb = sum(d.get("dram_read_bytes", 0.0) + d.get("dram_write_bytes", 0.0) for d in summary["kernels"]
                 if d.get("dram_read_bytes") == d.get("dram_read_bytes"))
        json.dump({"source": a.out + ".json", "kernels": [d["kernel"] for d in summary["kernels"]],
                   "dram_bytes_per_eval": tb, "note": a.note}, open(a.traffic_out, "w"), indent=1)
    open(a.out + ".md", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
