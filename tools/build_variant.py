"""Build an experiment variant of libgdgpu.so with extra -D flags into
paper_1506_04322_b200/_variants/libgdgpu_<name>.so; select it at run time with
GD_LIBRARY=<path>.  Usage: python tools/build_variant.py NAME -DGD_TRI_U=2 ..."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1506_04322_b200 import _build

name, defs = sys.argv[1], sys.argv[2:]
out = _build.PKG / "_variants"
print(_build.build(force=True, defines=defs, lib=out / f"libgdgpu_{name}.so",
                   objdir=out / f"obj_{name}"))
