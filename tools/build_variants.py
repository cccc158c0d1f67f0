"""Build library variants with extra -D defines into variants/ for A/B runs (FEA_LIB_PATH).

  python tools/build_variants.py name:-DX=1,-DY=2 name2:-DZ=3
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2012_00585_b200.build import build  # noqa: E402

out = Path(__file__).resolve().parents[1] / "variants"
out.mkdir(exist_ok=True)
for spec in sys.argv[1:]:
    name, _, defs = spec.partition(":")
    lib = out / f"libfea_{name}.so"
    build(force=True, out=lib, defines=tuple(d for d in defs.split(",") if d))
    print(lib)
