"""C-ABI library checks that need no GPU: it loads, exports every declared symbol, its host
logic (slab plan) is right, and the product package never touches the oracle."""
import ctypes
import os
import re

import pytest

from conftest import ROOT


def _header_functions():
    txt = open(os.path.join(ROOT, "include", "heatfem.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hf_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    import paper_1905_07622_b200 as hf
    lib = ctypes.CDLL(hf.LIB_PATH)
    names = _header_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # the Python binding exposes the same names
    assert sorted(hf.ABI_FUNCTIONS) == names
    for n in names:
        assert callable(getattr(hf, n))


def test_version_and_no_gpu_error_path():
    import paper_1905_07622_b200 as hf
    assert "sm_100a" in hf.hf_version()
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(hf.HfError) as e:
        hf.hf_create(((4, 4, 4), (1.0, 1.0, 1.0)), 0)
    assert e.value.status in (hf.HF_E_CUDA, hf.HF_E_OOM)


@pytest.mark.parametrize("nz1,nranks", [(100, 1), (100, 2), (101, 4), (512, 8), (17, 8), (2, 1)])
def test_slab_plan(nz1, nranks):
    import paper_1905_07622_b200 as hf
    ranges = [hf.hf_slab_plan(nz1, r, nranks) for r in range(nranks)]
    assert ranges[0][0] == 0 and ranges[-1][1] == nz1
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1 and min(sizes) >= 2


def test_slab_plan_errors():
    import paper_1905_07622_b200 as hf
    with pytest.raises(hf.HfError) as e:
        hf.hf_slab_plan(7, 0, 4)
    assert e.value.status == hf.HF_E_PARTITION
    with pytest.raises(hf.HfError) as e:
        hf.hf_slab_plan(100, 3, 2)
    assert e.value.status == hf.HF_E_ARG


def test_product_never_uses_oracle():
    pkg = os.path.join(ROOT, "paper_1905_07622_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), f
                assert "heat_oracle" not in src and "liboracle" not in src, f
                assert not re.search(r"^\s*(import|from)\s+synth\b", src, re.M), f
                assert not re.search(r"^\s*(import|from)\s+comparator\b", src, re.M), f
    # and the oracle never includes product code
    osrc = open(os.path.join(ROOT, "oracle", "heat_oracle.c")).read()
    includes = re.findall(r"^\s*#\s*include\s*[<\"]([^>\"]+)", osrc, re.M)
    assert includes and all(i in ("math.h", "omp.h", "stdint.h", "stdlib.h", "string.h") for i in includes), includes


def test_binding_rejects_bad_arrays():
    import numpy as np
    import paper_1905_07622_b200 as hf
    with pytest.raises(hf.HfError):
        hf._ptr(np.zeros(4, dtype=np.float32), 4)
    with pytest.raises(hf.HfError):
        hf._ptr(np.zeros(5), 4)
    with pytest.raises(hf.HfError):
        hf._ptr(np.zeros((4, 4))[:, 0], 4)
