"""C-ABI checks that need no GPU: libpd.so builds/loads, exports every function include/pd.h
declares, and rejects bad arguments before touching the device."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2605_06408_b200 as pd
from paper_2605_06408_b200 import build as pdbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "pd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pd_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    pdbuild.build()
    return pd.load_library()


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) <= set(pd.EXPORTED) | set(names)
    assert lib.pd_abi_version() == 1


def test_rejects_bad_arguments_without_gpu(lib):
    pts = np.zeros((4, 3), np.float32)
    with pytest.raises(pd.PdError) as e:
        pd.build_diagram(np.zeros((0, 3), np.float32), None, (0, 0, 0, 1, 1, 1))
    assert e.value.status == pd.PD_EEMPTY
    with pytest.raises(pd.PdError) as e:
        pd.build_diagram(pts, None, (0, 0, 0, 1, 0, 1))
    assert e.value.status == pd.PD_EINVAL
    with pytest.raises(pd.PdError) as e:
        pd.build_diagram(pts, None, (0, 0, 0, 1, 1, 1), leaf_size=33)
    assert e.value.status == pd.PD_EINVAL
    assert lib.pd_strerror(3) == b"non-finite coordinate or weight"


def test_sm100a_cubin(lib):
    """The library carries sm_100a SASS (no PTX-JIT or other-arch fallback)."""
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", pd.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
