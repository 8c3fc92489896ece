"""The C-ABI library loads (no GPU needed) and exports every symbol the header declares;
ctypes struct layouts match the C compiler's."""
import ctypes
import os
import re
import subprocess
import tempfile

from paper_2403_17017_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "kernelpick_b200.h")


def declared():
    return re.findall(r"^KP_API [^\n(]*?\b(kp_\w+)\(", open(HDR).read(), flags=re.M)


def test_header_declares_exports():
    assert sorted(declared()) == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    for name in declared():
        assert hasattr(L, name), name
    assert L.kp_version().decode().startswith("kpb200")
    assert L.kp_reduce_workspace_bytes() > 0


def test_struct_layouts_match_c():
    src = f'#include "{HDR}"\n#include <stdio.h>\n#include <stddef.h>\nint main(){{' \
          'printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(kp_csr), sizeof(kp_outcome), sizeof(kp_prepared),' \
          'sizeof(kp_tree_header), sizeof(kp_tree_node), offsetof(kp_outcome, kernel));}\n'
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "s.c"), os.path.join(d, "s")
        open(c, "w").write(src)
        gcc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
        subprocess.run([gcc, "-o", exe, c], check=True)
        got = [int(v) for v in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    want = [ctypes.sizeof(_lib.kp_csr), ctypes.sizeof(_lib.kp_outcome), ctypes.sizeof(_lib.kp_prepared), 16, 24,
            _lib.kp_outcome.kernel.offset]
    assert got == want


def test_invalid_args_rejected_without_gpu():
    L = _lib.load()
    # divisor <= 0 is rejected before any device work
    assert L.kp_wave_ceil_max_sum(None, 1, 5, 0, 1, None, None, None) == _lib.KP_EINVAL
    assert L.kp_gather_features(None, 1, 0, 1, None, None, None) == _lib.KP_EINVAL
    A = _lib.kp_csr(10, 10, 5, 7, 0, 0, 0, 0)  # bad off_type
    n = ctypes.c_size_t()
    assert L.kp_prepare_bytes(0, ctypes.byref(A), 0, ctypes.byref(n)) == _lib.KP_EINVAL


def test_product_fails_loudly_without_gpu():
    import pytest
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2403_17017_b200 import _kernels
    with pytest.raises(_lib.BackendUnavailable):
        _kernels.length_stats([0, 1, 2])
