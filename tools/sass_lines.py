"""Per-source-line instruction counts and stall samples from an ncu report (experiment tool).

    python tools/sass_lines.py report.ncu-rep lib.so kernel-mangled-substring [top] [ncu-kernel-regex] [column]

column: the per-instruction metric to aggregate instead of "Instructions Executed" (e.g.
"L1 Wavefronts Shared Excessive" for shared-memory bank conflicts).

Exports the report's SASS page, disassembles the same kernel from the library with line info
(nvdisasm -g), maps SASS offsets to (file, line) and aggregates executed warp instructions and
stall samples per line.
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile


def main():
    rep, lib, kname = sys.argv[1], sys.argv[2], sys.argv[3]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    demangled = sys.argv[5] if len(sys.argv) > 5 else None
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
    out = subprocess.run(cmd, capture_output=True, text=True).stdout
    # one section per profiled launch: keep the first one whose kernel name matches
    sections = [sec for sec in out.split('"Kernel Name"')[1:]]
    pick = sections[0]
    if demangled:
        for sec in sections:
            if re.search(demangled, sec.splitlines()[0]):
                pick = sec
                break
    rows = list(csv.reader(io.StringIO('"Kernel Name"' + pick)))
    hdr = rows[1]
    ia = hdr.index(sys.argv[6] if len(sys.argv) > 6 else "Instructions Executed")
    isamp = hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[2:] if len(r) > ia and r[0].startswith("0x")]
    base = int(data[0][0], 16)
    cnt = {int(r[0], 16) - base: (float(r[ia] or 0), float(r[isamp] or 0)) for r in data}
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
    sass = ""
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        s = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
        if any(l.startswith(".text.") and kname in l for l in s.splitlines()):
            sass = s
            break
    lines = sass.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and kname in l)
    cur = ("?", 0)
    per = collections.defaultdict(lambda: [0.0, 0.0])
    for l in lines[start + 1:]:
        if l.startswith(".text.") or l.startswith("//----"):
            break
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
        if m:
            off = int(m.group(1), 16)
            if off in cnt:
                per[cur][0] += cnt[off][0]
                per[cur][1] += cnt[off][1]
    tot = sum(v[0] for v in per.values())
    stot = sum(v[1] for v in per.values())
    src_cache = {}

    def src(f, n):
        for d in ("paper_2605_26461_b200/csrc", "include"):
            p = os.path.join(d, f)
            if os.path.exists(p):
                src_cache.setdefault(p, open(p).read().splitlines())
                return src_cache[p][n - 1].strip() if n - 1 < len(src_cache[p]) else ""
        return ""

    print(f"total warp inst {tot:.0f}  samples {stot:.0f}")
    for (f, n), (c, s) in sorted(per.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * c / tot:5.1f}% inst {100 * s / max(stot, 1):5.1f}% smp  {f}:{n:<5} {src(f, n)[:90]}")


if __name__ == "__main__":
    main()
