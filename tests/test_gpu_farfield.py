"""Far field of the boundary term: the
solid-harmonic expansion of closed net-boundary cycles (and of edge slivers
closed by their chords) against the exact fan sum (GWN_FARFIELD=0 switches the expansion off at scene creation), in fresh
processes so the switch is read at library load."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# the far field's guaranteed bound on |dw| per query (kFFDw, gwn_farfield.cuh:
# every expanded entry's truncation <= 2 pi kFFDw / entries); measured
# differences against the exact sum are 2e-12 (config 5) to 4e-11 (config 3)
# with the order thresholds taken from the computed moments
FF_DW = 1e-8

_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
cfg, nq, out, mode = int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
s = scenes.make(cfg, nq)
sc = G.Scene(s.ctrl)
q = s.queries
if mode == "far":  # single patch, queries 8..40 patch radii away
    rng = np.random.default_rng(0)
    c = s.ctrl.reshape(-1, 3).mean(0)
    u = rng.normal(size=(1024, 3)); u /= np.linalg.norm(u, axis=1)[:, None]
    q = c + np.repeat([8.0, 12.0, 20.0, 40.0], 256)[:, None] * u
if mode == "raypts":  # 64 rays x 100 points across the scene box (few far pairs per bucket)
    rng = np.random.default_rng(101)
    lo, hi = s.ctrl.reshape(-1, 3).min(0), s.ctrl.reshape(-1, 3).max(0)
    org = lo + rng.uniform(size=(64, 3)) * (hi - lo)
    d = rng.normal(size=3); d /= np.linalg.norm(d)
    span = np.linalg.norm(hi - lo)
    ts = np.sort(rng.uniform(-0.5 * span, 0.5 * span, size=(64, 100)), axis=1).ravel()
    q = np.repeat(org, 100, axis=0) + ts[:, None] * d[None, :]
qd = torch.from_numpy(np.ascontiguousarray(q)).cuda()
w, st = G.winding_numbers(sc, qd)
extra = {}
if mode == "halves":  # the same queries in two calls with global index bases
    h = len(q) // 2
    w1, s1 = G.winding_numbers(sc, qd[:h], index_base=0)
    w2, s2 = G.winding_numbers(sc, qd[h:], index_base=h)
    extra = dict(wh=torch.cat([w1, w2]).cpu().numpy(), sh=torch.cat([s1, s2]).cpu().numpy())
np.savez(out, w=w.cpu().numpy(), st=st.cpu().numpy(), far=sc.stats()["far_pairs"],
         shadow=sc.stats()["shadow_pairs"], near=sc.stats()["near_pairs"],
         cycles=sc.n_far_cycles, local=sc.stats()["local_evals"],
         levels=sc.local_expansions["levels"], **extra)
"""


def _run(tmp_path, cfg, nq, mode="plain", **env):
    tag = "_".join(f"{k}{v}" for k, v in sorted(env.items()))
    f = str(tmp_path / f"r{cfg}_{nq}_{mode}_{tag}.npz")
    e = dict(os.environ, **env)
    subprocess.run([sys.executable, "-c", _SCRIPT, REPO, str(cfg), str(nq), f, mode], env=e,
                   check=True, timeout=600)
    with np.load(f) as z:
        return {k: z[k] for k in z.files}


def test_farfield_matches_exact_sum_config5(tmp_path):
    ex = _run(tmp_path, 5, 1 << 13, GWN_FARFIELD="0")
    ff = _run(tmp_path, 5, 1 << 13)
    assert int(ex["cycles"]) == 0 and int(ff["cycles"]) > 100
    assert int(ff["far"]) > 0
    assert np.array_equal(ex["st"], ff["st"])
    ok = ex["st"] == 0
    assert np.abs(ex["w"] - ff["w"])[ok].max() <= FF_DW


def test_shadow_pairs_match_exact_sum_config5(tmp_path):
    """Pairs whose forward half-line crosses a cycle's sphere (the sphere in
    front of the query, beyond R_min) are far when their cell of the cycle's
    shadow winding grid is clean: expansion + 2 pi x winding number (DESIGN
    §9 f4).  A wrong winding number or sign would move w by 1/2 or more; the
    exact sum's status flags (band, degenerate) must be unchanged."""
    n = 1 << 15
    ex = _run(tmp_path, 5, n, GWN_FARFIELD="0")
    ff = _run(tmp_path, 5, n)
    assert int(ff["shadow"]) > n // 4          # the path is exercised
    assert int(ff["near"]) < int(ff["far"]) // 2
    assert np.array_equal(ex["st"], ff["st"])
    ok = ex["st"] == 0
    assert np.abs(ex["w"] - ff["w"])[ok].max() <= FF_DW


def test_local_expansions_match_per_pair_far_field_and_exact_config5(tmp_path):
    """Round 0's octree of local expansions (gwn_fmm.cu) against the per-pair
    far field (GWN_FMM=0) and the exact sum (GWN_FARFIELD=0): each translated
    (box, cycle) pair carries the per-pair path's bound."""
    n = 1 << 14
    ex = _run(tmp_path, 5, n, GWN_FARFIELD="0")
    pp = _run(tmp_path, 5, n, GWN_FMM="0")
    fm = _run(tmp_path, 5, n)
    assert int(pp["levels"]) == 0 and int(pp["local"]) == 0
    assert int(fm["levels"]) >= 2 and int(fm["local"]) >= n - 64  # queries inside the cube
    assert int(fm["far"]) < int(pp["far"]) // 10   # most cycles came from the expansions
    assert np.array_equal(ex["st"], fm["st"]) and np.array_equal(pp["st"], fm["st"])
    ok = ex["st"] == 0
    assert np.abs(fm["w"] - pp["w"])[ok].max() <= FF_DW
    assert np.abs(fm["w"] - ex["w"])[ok].max() <= FF_DW


def test_farfield_far_queries_single_cycle(tmp_path):
    ex = _run(tmp_path, 1, 16, mode="far", GWN_FARFIELD="0")
    ff = _run(tmp_path, 1, 16, mode="far", GWN_FF_ALL="1")
    assert int(ff["cycles"]) == 1 and int(ff["far"]) == 1024
    assert np.abs(ex["w"] - ff["w"]).max() <= FF_DW


def test_farfield_batching_is_bit_identical(tmp_path):
    r = _run(tmp_path, 5, 1 << 12, mode="halves")
    assert int(r["far"]) > 0
    assert np.array_equal(r["w"], r["wh"]) and np.array_equal(r["st"], r["sh"])


def test_single_patch_border(tmp_path):
    """Config 1: one open patch whose border cycle is expanded as edge slivers
    closed by their chords (the chord's exact fan term added back) once the
    budget allows it: the far pairs stay within the far-field bound of the
    exact sum, with identical statuses."""
    ex = _run(tmp_path, 1, 1 << 12, GWN_FARFIELD="0")
    ff = _run(tmp_path, 1, 1 << 12)
    assert np.array_equal(ex["st"], ff["st"])
    ok = ex["st"] == 0
    assert np.abs(ex["w"] - ff["w"])[ok].max() <= FF_DW


def test_small_far_buckets_config1(tmp_path):
    """Far pairs are evaluated bucket by bucket ((order level, entry) keys).
    With four entries and a few thousand far pairs a 128-record block spans
    several buckets and can begin and end in the same entry: it must not
    evaluate the records in between with that entry's moments (regression:
    4.5e-4 on these points)."""
    ex = _run(tmp_path, 1, 16, mode="raypts", GWN_FARFIELD="0")
    ff = _run(tmp_path, 1, 16, mode="raypts")
    assert int(ff["far"]) > 1000
    assert np.array_equal(ex["st"], ff["st"])
    ok = ex["st"] == 0
    assert np.abs(ex["w"] - ff["w"])[ok].max() <= FF_DW


def test_open_sheet_edge_slivers(tmp_path):
    """Config 3: the border cycle is too large to be far, so each of its 32
    edges is expanded as a sliver closed by its chord (the chord's exact fan
    term added back)."""
    ex = _run(tmp_path, 3, 1 << 14, GWN_FARFIELD="0")
    ff = _run(tmp_path, 3, 1 << 14)
    assert int(ff["cycles"]) == 32 and int(ff["far"]) > 0
    assert np.array_equal(ex["st"], ff["st"])
    ok = ex["st"] == 0
    assert np.abs(ex["w"] - ff["w"])[ok].max() <= FF_DW
