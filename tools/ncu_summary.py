"""Summarise an ncu --set full report: per-kernel key metrics, top stall reasons and the
hottest CUDA source lines (needs -lineinfo).  Usage:
    python tools/ncu_summary.py report.ncu-rep [kernel-regex] [--json out.json]"""

import csv
import io
import json
import re
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sectors_srcunit_tex_op_read.sum",
        "lts__t_sector_hit_rate.pct"]


def ncu(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu(["-i", rep, "--page", "raw", "--csv"]))))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for k in KEYS:
            if k in hdr:
                d[k] = (r[hdr.index(k)] + " " + units[hdr.index(k)]).strip()
        st = {h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(r[i] or 0)
              for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
              and h.endswith("per_issue_active.ratio")}
        d["stalls"] = dict(sorted(st.items(), key=lambda x: -x[1])[:6])
        out.append(d)
    return out


def hot_lines(rep, kregex, top=15):
    txt = ncu(["-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kregex}"])
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = None
    agg = {}
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            si = hdr.index("Warp Stall Sampling (All Samples)")
            continue
        if hdr is None or len(r) < len(hdr) or r[0] in ("-", ""):
            continue
        try:
            agg[(int(r[0]), r[1].strip()[:90])] = agg.get((int(r[0]), r[1].strip()[:90]), 0) + int(r[si] or 0)
        except ValueError:
            pass
    tot = sum(agg.values()) or 1
    return [(round(100 * v / tot, 1), k[0], k[1]) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]]


def main():
    rep = sys.argv[1]
    kre = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
    res = {"kernels": raw(rep)}
    if kre:
        res["hot_lines"] = hot_lines(rep, kre)
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
    for k in res["kernels"]:
        print("==", k["kernel"])
        for a, b in k.items():
            if a not in ("kernel", "stalls"):
                print(f"   {a:70s} {b}")
        print("   stalls:", k["stalls"])
    for h in res.get("hot_lines", []):
        print(f"  {h[0]:5.1f}%  L{h[1]:4d}  {h[2]}")


if __name__ == "__main__":
    main()
