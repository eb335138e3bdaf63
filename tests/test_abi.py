"""CPU checks of the C-ABI boundary: the library builds, loads, exports every symbol include/tawpipe.h
declares, and reports errors without a GPU.  No compute calls are made here."""
import os
import re

import pytest

from helpers import ROOT


def header_functions():
    with open(os.path.join(ROOT, "include", "tawpipe.h")) as fh:
        txt = fh.read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(tawpipe_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def L():
    from paper_2511_09741_b200 import build, tawpipe
    build.build()
    return tawpipe.lib()


def test_header_declares_the_north_star_calls():
    fns = header_functions()
    for f in ("tawpipe_init", "tawpipe_step", "tawpipe_shard"):
        assert f in fns


def test_every_declared_symbol_is_exported(L):
    missing = [f for f in header_functions() if not hasattr(L, f)]
    assert not missing, missing


def test_errors_before_init(L):
    from paper_2511_09741_b200 import tawpipe as T
    assert L.tawpipe_init(1, 1, 2, None, 1) == T.EUNINIT
    assert "bootstrap" in T.last_error()
    assert L.tawpipe_shard_elems() == T.EUNINIT
    import math
    assert math.isnan(L.tawpipe_step(None))
    assert L.tawpipe_trace_json(None, 0) == T.EUNINIT
    assert L.tawpipe_set_link_emulation(1.25, 30.0, 2) == T.EUNINIT


def test_unique_id_without_gpu(L):
    from paper_2511_09741_b200 import tawpipe as T
    a, b = T.unique_id(), T.unique_id()
    assert len(a) == 128 and a != b


def test_dims_struct_matches_header_layout():
    import ctypes
    from paper_2511_09741_b200.tawpipe import Dims
    # 10 int32 + 7 float + (4 bytes padding) + uint64
    assert ctypes.sizeof(Dims) == 10 * 4 + 7 * 4 + 4 + 8
    assert Dims.seed.offset == 72
