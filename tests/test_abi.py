"""C-ABI checks that need no GPU: libqdt.so builds/loads and exports every symbol that
include/qdt.h declares; the binding's names match; the product package never touches oracle/."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "qdt.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qdt_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ["qdt_init", "qdt_finalize", "qdt_build_probes", "qdt_solve", "qdt_objective",
                 "qdt_probes_free", "qdt_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    import paper_2404_02844_b200 as q
    from paper_2404_02844_b200 import build as b
    b.build()
    lib = ctypes.CDLL(q.LIB_PATH)
    for name in _declared():
        assert hasattr(lib, name), name
    assert sorted(q.ABI_SYMBOLS) == _declared()


def test_no_cuda_device_is_a_loud_error():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2404_02844_b200 as q
    with pytest.raises(q.QdtError) as e:
        q.qdt_init(0)
    assert "QDT_ERR_CUDA" in str(e.value)


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2404_02844_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).lower().replace(
                    "oracle/", ""), f
    for f in ["bench.py"]:
        pass


def test_build_uses_sm100a():
    from paper_2404_02844_b200 import build as b
    cmd = " ".join(b.nvcc_cmd())
    assert "arch=compute_100a,code=sm_100a" in cmd and "-lineinfo" in cmd
