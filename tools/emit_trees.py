"""Emit the frozen Seer bundle as one C/CUDA header: the three trees as
nested conditionals plus seer_dispatch, infer's control flow.
libkpb200 compiles it into the plan's selection kernel (kp_reduce.cu); plain-C hosts
include it directly.

    python tools/emit_trees.py [bundle.json] [out.h]      (default: include/kp_seer_trees.h)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_17017_b200 import seer  # noqa: E402

BUNDLE = os.path.join(ROOT, "paper_2403_17017_b200", "models", "seer_b200.json")
HEADER = os.path.join(ROOT, "include", "kp_seer_trees.h")


def render(bundle: str = BUNDLE) -> str:
    return seer.SeerModel.load(bundle).emit_header(os.path.relpath(bundle, ROOT))


if __name__ == "__main__":
    src = sys.argv[1] if len(sys.argv) > 1 else BUNDLE
    dst = sys.argv[2] if len(sys.argv) > 2 else HEADER
    with open(dst, "w") as f:
        f.write(render(src))
    print(dst)
