"""Experiment build: python tools/expbuild.py NAME [-DFOO=1 ...] -> exp/NAME/libhdll_b200.so

Objects of the shipped build are reused (copied) except for the sources named
by --redo=a.cu,b.cu (default: all), which are recompiled with the defines.
"""
import shutil, sys
from pathlib import Path
sys.path.insert(0, ".")
from paper_2309_11072_b200 import _build as B

name = sys.argv[1]
defs = [a[2:] for a in sys.argv[2:] if a.startswith("-D")]
redo = [a.split("=", 1)[1].split(",") for a in sys.argv[2:] if a.startswith("--redo=")]
out = Path("exp") / name
out.mkdir(parents=True, exist_ok=True)
B.build()  # the shipped objects are current
if redo:
    for o in B.BUILD.glob("*.o"):
        if o.stem + ".cu" not in redo[0]:
            shutil.copy2(o, out / o.name)
    for r in redo[0]:
        (out / (Path(r).stem + ".o")).unlink(missing_ok=True)
print(B.build(defines=defs, lib=out / "libhdll_b200.so", objdir=out))
