"""Emitted trees: include/kp_seer_trees.h is the frozen bundle's
emit_header, and its C text (the same text libkpb200 compiles into the plan's selection
kernel) answers exactly as DecisionTree.predict / SeerModel.predict_host -- checked here by
compiling it with gcc and running it on random vectors plus every threshold exactly."""
import os
import subprocess
import tempfile

import numpy as np

from paper_2403_17017_b200 import _lib, seer

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUNDLE = os.path.join(ROOT, "paper_2403_17017_b200", "models", "seer_b200.json")
HEADER = os.path.join(ROOT, "include", "kp_seer_trees.h")


def _model():
    return seer.SeerModel.load(BUNDLE)


def vectors(model, n=20_000, seed=5):
    """(n, 8) feature vectors: log-uniform known features, density-like gathered ones, and
    one row per internal node of every tree with that node's feature set exactly to its
    threshold (the `<=` boundary)."""
    rng = np.random.default_rng(seed)
    X = np.empty((n, 8))
    X[:, 0] = np.exp(rng.uniform(0, np.log(1e8), n))
    X[:, 1] = np.where(rng.random(n) < 0.7, X[:, 0], np.exp(rng.uniform(0, np.log(1e8), n)))
    X[:, 2] = X[:, 0] * np.exp(rng.uniform(0, np.log(2000), n))
    X[:, 3] = rng.choice([1, 2, 3, 5, 7, 10, 30, 64, 65, 100, 1000], n)
    X[:, 4] = 10 ** rng.uniform(-8, 0, n)
    X[:, 5] = X[:, 4] * rng.random(n)
    X[:, 6] = (X[:, 4] + X[:, 5]) / 2
    X[:, 7] = 10 ** rng.uniform(-16, -2, n)
    X[:, :4] = np.maximum(np.round(X[:, :4]), 1)
    hits = []
    for t in (model.selector_tree, model.known_tree, model.gathered_tree):
        for i in range(t.n_nodes):
            if t.feature[i] >= 0:
                row = X[len(hits) % n].copy()
                row[t.feature[i]] = t.threshold[i]
                hits.append(row)
    return np.vstack([X, np.array(hits)])


def test_header_is_the_bundle():
    """The committed header is exactly what tools/emit_trees.py renders from the bundle."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("emit_trees", os.path.join(ROOT, "tools", "emit_trees.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    assert open(HEADER).read() == mod.render(BUNDLE), "include/kp_seer_trees.h is stale: run tools/emit_trees.py"
    m = _model()
    import hashlib
    sha = hashlib.sha256(m.selector_tree.pack() + m.known_tree.pack() + m.gathered_tree.pack()).hexdigest()
    assert f'KP_SEER_TREES_SHA256 "{sha}"' in open(HEADER).read()
    # the library was built from this header
    assert _lib.load().kp_seer_emitted_sha256().decode() == sha


def test_emitted_header_matches_predict_host():
    m = _model()
    X = vectors(m)
    src = f'''#include <stdio.h>
#include "{HEADER}"
int main(void) {{
    double v[8];
    while (fread(v, sizeof(double), 8, stdin) == 8) {{
        int path = -7;
        int k = seer_dispatch(v[0], v[1], v[2], v[3], v + 4, &path);
        int kn = seer_dispatch(v[0], v[1], v[2], v[3], NULL, NULL);
        printf("%d %d %d %d %d %d %d\\n", seer_selector(v), seer_known(v), seer_gathered(v), k, path, kn,
               seer_needs_gathered(v[0], v[1], v[2], v[3]));
    }}
    return 0;
}}
'''
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "e.c"), os.path.join(d, "e")
        open(c, "w").write(src)
        gcc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
        subprocess.run([gcc, "-std=c99", "-O2", "-Wall", "-Werror", "-o", exe, c], check=True)
        out = subprocess.run([exe], input=X.astype("<f8").tobytes(), capture_output=True, check=True).stdout
    got = np.array([[int(t) for t in ln.split()] for ln in out.decode().splitlines()])
    assert got.shape == (X.shape[0], 7)
    for i, v in enumerate(X):
        kv, g = tuple(v[:4]), tuple(v[4:])
        kern, path = m.predict_host(*kv, g)
        want = (m.selector_tree.predict(kv), m.known_tree.predict(kv), m.gathered_tree.predict(tuple(v)),
                kern, path, kern if path == seer.USE_KNOWN else -1, path)
        assert tuple(got[i]) == want, (i, v, got[i], want)
