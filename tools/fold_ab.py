"""A/B timing of the fold across library builds: python tools/fold_ab.py lib1.so lib2.so ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "one":
    os.environ["MPSF_LIB"] = sys.argv[2]
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fold_run.py"), "30"], capture_output=True,
                         text=True, env=os.environ)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
    import ast
    try:
        d = ast.literal_eval(line)
        print(round(d["ms_per_step"] * 1e3, 1), "us", d["bit_exact_vs_oracle"])
    except Exception:
        print(line)
else:
    for lib in sys.argv[1:]:
        r = subprocess.run([sys.executable, __file__, "one", lib], capture_output=True, text=True)
        print(os.path.basename(lib), r.stdout.strip() or r.stderr[-300:], flush=True)
