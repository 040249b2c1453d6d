"""CPU: the C-ABI library loads, exports every symbol include/mscg.h
declares, fails loudly without a GPU, and the product never reaches into
oracle/."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exports_every_declared_symbol(msc):
    from paper_1104_3349_b200 import _capi
    L = _capi.lib()
    declared = _capi.declared_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if not hasattr(L, s)]
    assert missing == []
    # and the Python binding covers all of them with signatures
    assert sorted(_capi._SIGS) == declared
    assert L.mscg_abi_version() == 1


def test_no_gpu_fails_loudly(msc):
    from conftest import HAS_GPU
    if HAS_GPU:
        pytest.skip("GPU present")
    with pytest.raises(msc.CudaError, match="no CUDA device"):
        msc.Context(0)


def test_random_vector_matches_reference(msc, ref):
    from paper_1104_3349_b200 import _capi
    out = np.empty(1000)
    _capi.lib().mscg_random_vector(1000, 0, out.ctypes.data_as(C.c_void_p))
    assert np.array_equal(out, ref.random_vector(1000, 0))


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1104_3349_b200")
    pat = re.compile(r"\b(refpy|restatepy|oracle|libmscref|liborestate)\b")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".hpp", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                hits = [ln for ln in src.splitlines()
                        if pat.search(ln) and not ln.lstrip().startswith(("//", "#", "*"))]
                assert hits == [], (f, hits)


def test_header_functions_are_extern_c():
    src = open(os.path.join(ROOT, "include", "mscg.h")).read()
    assert 'extern "C"' in src and "MSCG_ABI_VERSION" in src
