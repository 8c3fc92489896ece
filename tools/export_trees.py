"""Export the frozen Seer bundle's three trees in the packed C-ABI layout for hosts that
do not read JSON (examples/seer_run.c).  File: b"KPT1" then, for selector, known,
gathered: uint32 byte count + kp_tree_header/kp_tree_node bytes (dtree.pack, little endian).

    python tools/export_trees.py [bundle.json] [out.trees]"""
import os
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_17017_b200 import seer  # noqa: E402

src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2403_17017_b200", "models", "seer_b200.json")
dst = sys.argv[2] if len(sys.argv) > 2 else os.path.splitext(src)[0] + ".trees"
m = seer.SeerModel.load(src)
with open(dst, "wb") as f:
    f.write(b"KPT1")
    for t in (m.selector_tree, m.known_tree, m.gathered_tree):
        b = t.pack()
        f.write(struct.pack("<I", len(b)))
        f.write(b)
print(dst)
