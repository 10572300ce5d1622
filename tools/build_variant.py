"""Experiment builds: compile the library with extra nvcc flags into
paper_2301_01356_b200/_variants/<name>.so (git-ignored, travels to the GPU
box); select one at run time with FBCC_LIB=<path>.
    python tools/build_variant.py NAME -DFOO=1 ..."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2301_01356_b200 import build  # noqa: E402

if __name__ == "__main__":
    name, flags = sys.argv[1], sys.argv[2:]
    out = build.PKG / "_variants" / f"{name}.so"
    print(build.build(extra=flags, out=out))
