#!/usr/bin/env python3
"""A/B timing of libgb builds (GPU box): for every ab/*.so (built here with
`python -m paper_2603_02621_b200.build -D ... -o ab/<name>.so`) plus the default
libgb.so, run scripts/prof_one.py --time in a fresh process with GB_LIB set, and
print each build's median launch time and result digest (must agree).

usage: python scripts/ab_time.py [--span 36] [--N 1e12] [--reps 10]
"""
import argparse
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--span", type=int, default=36)
ap.add_argument("--N", default="1e12")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--rounds", type=int, default=2)
ap.add_argument("--abdir", default="ab", help="directory of the A/B builds")
ap.add_argument("--hi", default=None, help="exclusive top of the range (e.g. 4000000000000000000 for C5)")
a = ap.parse_args()
libs = [os.path.join(ROOT, "paper_2603_02621_b200", "libgb.so")] + sorted(glob.glob(os.path.join(ROOT, a.abdir, "*.so")))
for rnd in range(a.rounds):
    for lib in libs:
        env = dict(os.environ, GB_LIB=lib)
        r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "prof_one.py"), "--span", str(a.span),
                            "--N", a.N, "--time", str(a.reps)] + (["--hi", a.hi] if a.hi else []), env=env, capture_output=True, text=True)
        lines = [l for l in r.stdout.splitlines() if l.startswith("{") or l.startswith("TIME")]
        print(os.path.basename(lib), r.returncode, " | ".join(lines), r.stderr[-300:] if r.returncode else "",
              flush=True)
