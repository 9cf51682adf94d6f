"""A/B variants of libpd.so built with extra -D defines (tuning knobs), timed with tools/quick_perf.py.

    python tools/ab.py build NAME DEF1 DEF2 ...     (here: cross-compile paper_2605_06408_b200/libpd_NAME.so)
    python tools/ab.py run NAME [configs...]        (GPU box: PD_LIB=... quick_perf)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if sys.argv[1] == "build":
    from paper_2605_06408_b200 import build as b
    name = sys.argv[2]
    out = os.path.join(ROOT, "paper_2605_06408_b200", f"libpd_{name}.so")
    b.build(force=True, defines=tuple(sys.argv[3:]), out=out)
    print(out)
else:
    name = sys.argv[2]
    lib = os.path.join(ROOT, "paper_2605_06408_b200", "libpd.so" if name == "base" else f"libpd_{name}.so")
    env = dict(os.environ, PD_LIB=lib)
    cfgs = sys.argv[3:] or ["C4"]
    print("==", name, flush=True)
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "quick_perf.py")] + cfgs, env=env, check=False)
