"""A/B timing of experiment builds: python tools/ab.py NIMG CONFIG ROUNDS STEPS lib1.so lib2.so ...

Each round runs tools/steptimes.py once per library (HDLL_B200_LIB), in turn,
so the variants interleave on one box; prints the median step and stage times
per library over every round's steps after the first of each run.
"""
import json, os, subprocess, sys
from collections import defaultdict
from statistics import median

nimg, cfg, rounds, steps = sys.argv[1:5]
libs = sys.argv[5:]
res = defaultdict(lambda: defaultdict(list))
for r in range(int(rounds)):
    for lib in libs:  # "path.so[,VAR=VALUE...]"
        path, *kv = lib.split(",")
        env = dict(os.environ, HDLL_B200_LIB=os.path.abspath(path), **dict(a.split("=", 1) for a in kv))
        out = subprocess.run([sys.executable, "tools/steptimes.py", nimg, cfg, steps], env=env,
                             capture_output=True, text=True)
        lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
        if not lines or out.returncode:
            print(lib, "FAILED", out.stderr[-800:], flush=True)
            continue
        for l in lines[1:]:
            if l["rc"] != 0:
                print(lib, "rc", l["rc"], flush=True)
            res[lib]["step"].append(l["ms"])
            for k, v in l["stages"].items():
                res[lib][k].append(v)
for lib in libs:
    d = res[lib]
    print(lib, " ".join(f"{k}={median(v):.3f}" for k, v in d.items() if v), flush=True)
