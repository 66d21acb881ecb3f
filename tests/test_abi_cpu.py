"""Host-side checks of the C-ABI library (no GPU needed): it builds for sm_100a,
loads, exports every symbol include/pcdm.h declares, the binding covers them,
and argument validation that happens before any CUDA call behaves."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_1212_0873_b200 import build, pcdm
    build.build()
    return pcdm.load()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "pcdm.h")).read()
    return sorted(set(re.findall(r"PCDM_API[^;(]*?\b(pcdm_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    syms = header_symbols()
    for s in ("pcdm_create", "pcdm_omega", "pcdm_run", "pcdm_objective"):
        assert s in syms


def test_library_exports_every_header_symbol(lib):
    from paper_1212_0873_b200 import pcdm
    out = subprocess.check_output(["nm", "-D", "--defined-only", pcdm.LIB_PATH]).decode()
    exported = set(re.findall(r"\sT\s(pcdm_\w+)", out))
    for s in header_symbols():
        assert s in exported, s
        assert hasattr(lib, s)
    assert sorted(pcdm.EXPORTS) == header_symbols()
    # nothing but the ABI is exported from our code
    assert exported == set(header_symbols())


def test_library_is_sm100a(lib):
    from paper_1212_0873_b200 import pcdm
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", pcdm.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_host_side_argument_validation(lib):
    from paper_1212_0873_b200 import pcdm
    c = np.array([0, 1], dtype=np.int64)
    r = np.array([0], dtype=np.int32)
    v = np.array([1.0], dtype=np.float32)
    b = np.array([1.0], dtype=np.float32)
    with pytest.raises(pcdm.PCDMError) as e:
        pcdm.pcdm_create(0, 1, c, r, v, b, 0.1, stream=0)
    assert e.value.status == pcdm.PCDM_EINVAL and "no loss terms" in e.value.message
    with pytest.raises(pcdm.PCDMError) as e:
        pcdm.pcdm_create(1, 1, c, r, v, b, -1.0, stream=0)
    assert e.value.status == pcdm.PCDM_EINVAL
    with pytest.raises(pcdm.PCDMError) as e:
        pcdm.pcdm_create(1, 1, c, r, v, b, float("nan"), stream=0)
    assert e.value.status == pcdm.PCDM_EINVAL
    with pytest.raises(pcdm.PCDMError) as e:
        pcdm.pcdm_sample(10, 11, 0, 0, 1, np.zeros(11, dtype=np.int32), stream=0)
    assert e.value.status == pcdm.PCDM_EINVAL
    with pytest.raises(TypeError):
        pcdm.pcdm_create(1, 1, c.astype(np.int32), r, v, b, 0.1, stream=0)


def test_binding_has_no_cpu_fallback():
    # the product package never imports the oracle
    pkg = os.path.join(ROOT, "paper_1212_0873_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "pcdm_oracle" not in txt, f
