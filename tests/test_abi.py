"""C-ABI library loads, exports every declared symbol, host helpers agree
with the oracle contract, and the product fails loudly without a GPU."""

import os
import re

import numpy as np
import pytest

from paper_2408_04466_b200 import _lib, engine, scenes
from oracle import oracle as O

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(REPO, "include", "gwn_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gwn_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    L = _lib.lib()
    names = _declared()
    assert len(names) >= 15
    for name in names:
        assert hasattr(L, name), name
    assert set(names) == set(_lib.EXPORTS)
    assert L.gwn_abi_version() == 6


def test_default_params_mirror_reference_epsilons():
    p = _lib.default_params()
    assert (p.residual, p.dedup, p.tangent, p.edge_graze, p.degenerate) == \
        (1e-10, 1e-9, 1e-12, 1e-10, 1e-12)
    assert p.samples_per_edge == 200 and p.max_rounds == 32 and p.max_jitters == 3


def test_direction_and_jitter_sequences_match_oracle():
    for r in range(40):
        assert np.array_equal(engine.direction(12345, r), O.direction(12345, r))
    import ctypes as C
    for q in (0, 1, 7, 1 << 40):
        for a in (1, 2, 3):
            v = np.empty(3)
            _lib.lib().gwn_jitter_dir(99, q, a, v.ctypes.data_as(C.POINTER(C.c_double)))
            assert np.array_equal(v, O.jitter_dir(99, q, a))


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_net_boundary_matches_oracle(cfg):
    ctrl = scenes.make(cfg, 4).ctrl
    e1, w1 = engine.net_boundary(ctrl)
    e2, w2 = O.net_boundary(ctrl)
    assert np.array_equal(e1, e2) and np.array_equal(w1, w2)


def test_scene_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2408_04466_b200.errors import DeviceError
    with pytest.raises(DeviceError):
        engine.Scene(scenes.make(1, 4).ctrl)


def test_scene_rejects_bad_input():
    from paper_2408_04466_b200.errors import SceneError
    with pytest.raises(SceneError):
        engine.Scene(np.zeros((2, 3, 4, 3)))
    with pytest.raises(ValueError):
        engine.Scene(np.zeros((1, 4, 4, 3)), samples_per_edge=1)
