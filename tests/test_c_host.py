"""The C-ABI driven from plain C (examples/seer_run.c): Matrix Market text -> kp_mm_parse
-> kp_csr_from_coo -> kp_seer_plan, no Python in the loop; its selection must equal the
Python host's on the same matrix, and the packed tree file must match the JSON bundle."""
import os
import struct
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODEL = os.path.join(ROOT, "paper_2403_17017_b200", "models", "seer_b200.json")
TREES = os.path.join(ROOT, "paper_2403_17017_b200", "models", "seer_b200.trees")


def test_packed_trees_match_bundle():
    from paper_2403_17017_b200 import seer
    m = seer.SeerModel.load(MODEL)
    b = open(TREES, "rb").read()
    assert b[:4] == b"KPT1"
    at = 4
    for t in (m.selector_tree, m.known_tree, m.gathered_tree):
        (n,) = struct.unpack_from("<I", b, at)
        at += 4
        assert b[at:at + n] == t.pack()
        at += n
    assert at == len(b)


@pytest.mark.gpu
@pytest.mark.parametrize("name,k", [("C1", 1), ("C4", 1), ("C3", 100)])
def test_c_host_matches_python_selection(tmp_path, name, k):
    import torch
    from paper_2403_17017_b200 import gen, mmio, seer
    exe = os.path.join(ROOT, "examples", "seer_run")
    if not os.path.exists(exe):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "examples")], check=True)
    m = gen.config(name, small=(name != "C1"))
    S = m.to_sparse_csr()
    mtx = tmp_path / f"{name}.mtx"
    mtx.write_text(mmio.write_matrix_market(S))
    out = subprocess.run([exe, str(mtx), TREES, str(k)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    kv = dict(p.split("=") for p in out.stdout.split())
    A = m.to_device_csr(torch.float64)
    o = seer.infer(seer.SeerModel.load(MODEL), A, k)
    assert (int(kv["kernel"]), int(kv["path"]), int(kv["nnz"])) == (o.chosen_kernel, o.path, A.nnz)
