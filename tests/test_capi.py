"""The C-ABI library (CPU-side checks, no GPU needed): it loads, exports every
function include/mca/mca_cuda.h declares, reports errors through status codes,
and the oracle's definitions satisfy the reference's own matrix.hpp."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mca", "mca_cuda.h")
REF_HEADER = "/root/reference/proj/include/mca/matrix.hpp"


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mca_[a-z_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2201_12854_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    return _lib.lib()


def test_header_and_binding_agree():
    from paper_2201_12854_b200 import _lib
    assert _declared_functions() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    from paper_2201_12854_b200 import _lib
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r" T (mca_\w+)", out))
    for name in _declared_functions():
        assert name in exported, name
        assert getattr(lib, name) is not None


def test_library_is_sm100a(lib):
    from paper_2201_12854_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_errors_are_status_codes_not_crashes(lib):
    from paper_2201_12854_b200 import _lib
    h = ctypes.c_void_p()
    # NULL weights -> MCA_ERR_NULL with a message, no exception crosses the ABI
    assert lib.mca_prepare_weights(None, 0, 768, 12, 64, None, ctypes.byref(h)) == _lib.MCA_ERR_NULL
    assert b"NULL" in lib.mca_last_error()
    cfg = _lib.McaConfigC(0.0, 0.0, 1, _lib.MCA_MODE_APPROX)   # alpha = 0 is rejected
    rc = lib.mca_stage_budgets(ctypes.c_void_p(8), 1, 4, 64, ctypes.byref(cfg), ctypes.c_void_p(8),
                               ctypes.c_void_p(8), None)
    assert rc == _lib.MCA_ERR_DOMAIN
    assert lib.mca_version().startswith(b"mca_b200")


def test_forward_attn_argument_errors(lib):
    """mca_forward_attn (the cli's device path) reports bad arguments as
    status codes before touching the device."""
    from paper_2201_12854_b200 import _lib
    cfg = _lib.McaConfigC(0.4, 0.0, 1, _lib.MCA_MODE_APPROX)
    rc = lib.mca_forward_attn(None, None, None, 0, 1, 16, 0, 0, ctypes.byref(cfg), 1, None, None, None, None, None)
    assert rc == _lib.MCA_ERR_NULL and b"weights" in lib.mca_last_error()
    bad = _lib.McaConfigC(1.5, 0.0, 1, _lib.MCA_MODE_APPROX)        # alpha outside (0, 1]
    rc = lib.mca_forward_attn(ctypes.c_void_p(8), None, None, 0, 1, 16, 0, 0, ctypes.byref(bad), 1, None, None, None,
                              None, None)
    assert rc == _lib.MCA_ERR_DOMAIN


def test_no_cuda_device_is_reported_loudly(lib):
    """On a host without a GPU the forward must fail loudly (MCA_ERR_CUDA),
    never fall back to a CPU computation."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2201_12854_b200 import _lib
    h = ctypes.c_void_p()
    rc = lib.mca_prepare_weights(ctypes.c_void_p(8), 0, 768, 12, 64, None, ctypes.byref(h))
    assert rc == _lib.MCA_ERR_CUDA
    assert b"no CUDA device" in lib.mca_last_error()


def test_python_api_refuses_cpu_tensors():
    import torch
    import paper_2201_12854_b200 as mca
    with pytest.raises(mca.CudaError):
        mca.AttentionWeights(torch.zeros(768, 768), heads=12)


@pytest.mark.skipif(not os.path.exists(REF_HEADER), reason="reference tree not mounted")
def test_oracle_satisfies_reference_header(tmp_path):
    """Compile oracle/tensor.cpp against the REFERENCE's matrix.hpp and link a
    client that uses every declared function: the declarations are the
    reference's, the definitions ours (oracle/Makefile `ref` target)."""
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    client = tmp_path / "client.cpp"
    client.write_text(
        '#include "mca/matrix.hpp"\n#include <cstdio>\nint main(){ using namespace mca;\n'
        'Matrix a = Matrix::from_rows({{1,2},{3,4}}), b(2,2,1.0);\n'
        'Matrix c = matmul(a,b), d = matmul_nt(a,b), t = transpose(a), s = softmax_rows(a, 1.0);\n'
        'auto r = row_l2_norms(a); auto k = col_l2_norms(a);\n'
        'double f = frobenius_norm(a) + col_max(a,1) + c.at(1,1) + d.at(0,0) + t.at(0,1) + s.at(0,0) + r[0] + k[1];\n'
        'std::printf("%d %.6f\\n", (int)a.all_finite(), f); return 0; }\n')
    exe = tmp_path / "client"
    subprocess.run(["/usr/bin/g++", "-std=c++20", "-I/root/reference/proj/include", str(client),
                    os.path.join(ROOT, "oracle", "_ref", "libmca_ref_tensor.so"), "-o", str(exe),
                    f"-Wl,-rpath,{os.path.join(ROOT, 'oracle', '_ref')}"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert out[0] == "1" and abs(float(out[1]) - 29.454371) < 1e-5


def test_torch_custom_op_registered_with_fake_kernel():
    """The PyTorch binding registers torch.ops.mca_b200.attention with a fake
    (meta) kernel: shape propagation works without a GPU (no library call)."""
    torch = pytest.importorskip("torch")
    from torch._subclasses.fake_tensor import FakeTensorMode
    import paper_2201_12854_b200.torch_op  # noqa: F401
    with FakeTensorMode():
        q = torch.empty(2, 16, 768)
        x = torch.empty(2, 16, 768)
        w = torch.empty(768, 768)
        y = torch.ops.mca_b200.attention(q, q, x, w, 12, 0.4, 0, "approximation", 0)
    assert tuple(y.shape) == (2, 16, 768)
