"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north star): integer classification exact away from the
surface, |dw| <= 1e-6 elsewhere.  We test tighter: closed scenes bit-exact,
open scenes |dw| <= 1e-9, on the same seeded inputs and global query ids.
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2408_04466_b200 as G  # noqa: E402
from paper_2408_04466_b200 import _kernels, scenes  # noqa: E402
from oracle import oracle as O  # noqa: E402

W_TOL = 1e-9     # open scenes, both statuses 0
SUB = {1: 4096, 2: 1 << 16, 3: 1 << 14, 4: 1 << 16, 5: 8192}
_cache = {}


def _scene(cfg, **kw):
    key = (cfg, tuple(sorted(kw.items())))
    if key not in _cache:
        s = scenes.make(cfg, SUB[cfg])
        _cache[key] = (s, G.Scene(s.ctrl, **kw))
    return _cache[key]


def _compare(cfg, w, st, wo, so):
    # same direction sequence and jitter hashes: the statuses agree query by
    # query (a borderline decision may differ on a handful)
    assert (st != so).sum() <= max(2, len(st) // 20000), (cfg, np.unique(st, return_counts=True),
                                                         np.unique(so, return_counts=True))
    both = (st == 0) & (so == 0)
    assert both.mean() > 0.995, (cfg, np.unique(st, return_counts=True),
                                 np.unique(so, return_counts=True))
    if cfg in (2, 4):
        assert np.array_equal(w[both], wo[both])
        assert np.all(w[both] == np.round(w[both]))
    else:
        d = np.abs(w - wo)[both]
        assert d.max() <= W_TOL, (cfg, d.max(), np.argmax(d))


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_config_parity_vs_oracle(cfg):
    s, sc = _scene(cfg)
    w, st = G.winding_numbers(sc, s.queries)
    wo, so, chi, rounds = O.scene_eval(s.ctrl, s.queries)
    _compare(cfg, w, st, wo, so)


def test_device_tensors_and_chunking_are_identical():
    s, sc = _scene(3)
    q = torch.from_numpy(s.queries).cuda()
    w, st = G.winding_numbers(sc, q)
    w2, st2 = G.winding_numbers(sc, s.queries)
    assert np.array_equal(w.cpu().numpy(), w2) and np.array_equal(st.cpu().numpy(), st2)
    sc_small = G.Scene(s.ctrl, chunk_queries=1000)
    w3, st3 = G.winding_numbers(sc_small, s.queries)
    assert np.array_equal(w3, w2) and np.array_equal(st3, st2)


@pytest.mark.parametrize("cfg", [2, 3])
def test_pipelined_host_path_equals_device_path(cfg):
    """Host buffers of >= 2^18 queries take the pipelined path (chunked input copies,
    rounds and output copies on three streams, tail chunk split): bit-identical to
    one device-resident eval, at an odd size."""
    s = scenes.make(cfg, (1 << 18) + 777)
    sc = G.Scene(s.ctrl)
    w, st = G.winding_numbers(sc, torch.from_numpy(s.queries).cuda())
    wh, sh = G.winding_numbers(sc, s.queries)
    assert np.array_equal(w.cpu().numpy(), wh) and np.array_equal(st.cpu().numpy(), sh)


def test_sharded_slices_equal_unsharded():
    s, sc = _scene(2)
    w, st = G.winding_numbers(sc, s.queries)
    n = len(s.queries)
    parts = [G.winding_numbers(sc, s.queries[a:b], index_base=a)
             for a, b in ((0, n // 3), (n // 3, n))]
    assert np.array_equal(np.concatenate([p[0] for p in parts]), w)
    assert np.array_equal(np.concatenate([p[1] for p in parts]), st)


def test_closed_cube_full_size_properties():
    s = scenes.make(2)                          # 1M queries, the bench config
    sc = G.Scene(s.ctrl)
    w, st = G.winding_numbers(sc, s.queries)
    ok = st == 0
    assert ok.mean() > 0.9999
    assert set(np.unique(w[ok])) <= {0.0, 1.0}
    r = np.linalg.norm(s.queries, axis=1)
    assert np.all(w[ok & (r < 0.75)] == 1.0) and np.all(w[ok & (r > 1.25)] == 0.0)
    # antisymmetry: flipped orientation negates w
    scf = G.Scene(np.swapaxes(s.ctrl, 1, 2))
    wf, stf = G.winding_numbers(scf, s.queries[: 1 << 18])
    m = ok[: 1 << 18] & (stf == 0)
    assert np.array_equal(wf[m], -w[: 1 << 18][m])


def test_north_star_full_size_properties():
    """BASELINE config 5 at its full size (15,876 patches, 2^26 queries): the
    8-GPU layout (eight query slices with global index bases, each a single
    chunk) gives the same bits as one call (two 2^25-query chunks); the far
    field's statistics are those of the bench; and flipping every patch's
    orientation negates w on a 2^22-query slice.  Oracle parity
    on a subsample of the same scene: test_config_parity_vs_oracle[5]."""
    s = scenes.make(5)
    n = len(s.queries)
    assert n == 1 << 26 and s.ctrl.shape[0] == 15876
    sc = G.Scene(s.ctrl)
    q = torch.from_numpy(s.queries).cuda()
    w, st = G.winding_numbers(sc, q)
    stt = sc.stats()
    assert stt["rounds"] >= 2 and stt["near_pairs"] < 1.5 * n < stt["far_pairs"]
    assert float((st == 0).double().mean()) > 0.9999
    assert bool(torch.isfinite(w).all()) and float(w.abs().max()) < 16.0
    per = n // 8
    for r in range(8):
        wr, sr = G.winding_numbers(sc, q[r * per:(r + 1) * per], index_base=r * per)
        assert torch.equal(wr, w[r * per:(r + 1) * per]) and torch.equal(sr, st[r * per:(r + 1) * per])
    del sc
    G.release_caches()
    scf = G.Scene(np.ascontiguousarray(np.swapaxes(s.ctrl, 1, 2)))
    m = 1 << 22
    wf, stf = G.winding_numbers(scf, q[:m])
    ok = (st[:m] == 0) & (stf == 0)
    assert float(ok.double().mean()) > 0.999
    assert float((wf + w[:m])[ok].abs().max()) <= W_TOL


def test_direction_independence_open_patch():
    s, sc = _scene(1)
    sc2 = G.Scene(s.ctrl, dir_seed=777)
    w1, s1 = G.winding_numbers(sc, s.queries)
    w2, s2 = G.winding_numbers(sc2, s.queries)
    m = (s1 == 0) & (s2 == 0)
    assert np.abs(w1 - w2)[m].max() < 1e-10


def test_rigid_invariance():
    s, _ = _scene(1)
    rng = np.random.default_rng(5)
    R = scenes.random_rotation(rng)
    t = rng.normal(size=3)
    a = G.Scene(s.ctrl)
    b = G.Scene(s.ctrl @ R.T + t)
    wa, sa = G.winding_numbers(a, s.queries)
    wb, sb = G.winding_numbers(b, s.queries @ R.T + t)
    m = (sa == 0) & (sb == 0)
    assert np.abs(wa - wb)[m].max() < 1e-9


def test_flipped_duplicate_cancels_and_additivity():
    s, _ = _scene(1)
    both = np.concatenate([s.ctrl, np.swapaxes(s.ctrl, 1, 2)])
    w, st = G.winding_numbers(G.Scene(both), s.queries)
    assert np.abs(w[st == 0]).max() < 1e-9
    # additivity over disjoint components
    c2 = scenes.make(2, 8).ctrl + np.array([5.0, 0, 0])
    wa, sa = G.winding_numbers(G.Scene(s.ctrl), s.queries)
    wb, sb = G.winding_numbers(G.Scene(c2), s.queries)
    wab, sab = G.winding_numbers(G.Scene(np.concatenate([s.ctrl, c2])), s.queries)
    m = (sa == 0) & (sb == 0) & (sab == 0)
    assert np.abs(wab - wa - wb)[m].max() < 1e-9


def test_spec_examples_and_edge_cases():
    flat = np.array([[(i / 3, j / 3, 0.0) for j in range(4)] for i in range(4)])
    p = G.BicubicPatch(flat)
    hits = p.all_hits(G.Ray(np.array([0.2, 0.2, 1.0]), np.array([0.0, 0.0, -1.0])))
    assert len(hits) == 1 and abs(hits[0].t - 1) < 1e-12 and hits[0].sign == -1
    assert p.all_hits(G.Ray(np.array([2.0, 2.0, 1.0]), np.array([0.0, 0.0, -1.0]))) == []
    sc = G.Scene([p], samples_per_edge=2000)
    w = G.winding_number(sc, [0.5, 0.5, 0.5])
    assert abs(w + 1 / 6) < 1e-6                 # code convention
    # empty batch, empty scene
    w0, s0 = G.winding_numbers(sc, np.zeros((0, 3)))
    assert w0.shape == (0,)
    we, se = G.winding_numbers(G.Scene(np.zeros((0, 4, 4, 3))), np.ones((5, 3)))
    assert np.all(we == 0) and np.all(se == 0)
    # query on the surface -> jittered, status 1; on a boundary vertex -> 3
    w1, s1 = G.winding_numbers(G.Scene([p]), np.array([[0.4, 0.6, 0.0], [0.0, 0.0, 0.0]]))
    assert s1[0] == 1 and s1[1] in (1, 3)


def test_all_hits_match_oracle_and_tessellation(golden_dir):
    r = np.load(os.path.join(golden_dir, "roots.npz"))
    for k in range(len(r["o"])):
        ctrl = r["ctrl"][r["pid"][k]]
        p = G.BicubicPatch(ctrl)
        gh = p.all_hits(G.Ray(r["o"][k], r["d"][k]))
        oh = O.patch_all_hits(ctrl, r["o"][k], r["d"][k])
        assert sum(h.sign for h in gh) == r["tess_chi"][k], k
        assert len(gh) == len(oh), k
        for a, b in zip(gh, oh):
            assert abs(a.t - b.t) < 1e-9 and a.sign == b.sign
            assert a.tangency == b.tangency and a.grazing == b.grazing


def test_single_loop_batch_matches_fixed_reference(golden_dir):
    f = np.load(os.path.join(golden_dir, "fan.npz"))
    for di in range(len(f["dirs"])):
        d = f["dirs"][di]
        for k in range(0, len(f["queries"]), 7):
            p = f["queries"][k]
            recs = O.patch_all_hits(f["ctrl"], p, d)
            ht = np.array([h.t for h in recs])
            hs = np.array([h.sign for h in recs], np.int64)
            w, ok = _kernels.single_loop_batch(f["loop"], p, d, ht, hs, np.zeros(1), 1e-9, 1e-12)
            assert ok[0] == 1
            if f["ok"][di, k]:
                assert abs(w[0] - f["w"][di, k]) < 1e-12
            else:
                assert abs(w[0] - (f["chi"][di, k] + O.loop_fan(f["loop"], p, d))) < 1e-12


def test_fp64_peak_measures():
    tf, ms = G.fp64_peak(0)
    assert 10.0 < tf < 60.0, tf


def test_k4_rsqrt_full_precision():
    import ctypes as C
    from paper_2408_04466_b200 import _lib
    u = C.c_uint64()
    _lib.check(_lib.lib().gwn_selftest_rsqrt(0, 1 << 20, C.byref(u)), "gwn_selftest_rsqrt")
    assert u.value <= 2, u.value


# ---------------------------------------------------------------------------
# edge cases the reference's degeneracy rules cover (errors.py)
# ---------------------------------------------------------------------------

def _edge_compare(ctrl, queries, tol=1e-9, min_ok=0.99, **kw):
    sc = G.Scene(ctrl, **kw)
    w, st = G.winding_numbers(sc, queries)
    prm = O.params(samples_per_edge=kw.get("samples_per_edge", 200))
    wo, so, _, _ = O.scene_eval(ctrl, queries, prm=prm)
    both = (st == 0) & (so == 0)
    assert both.mean() >= min_ok, (np.unique(st, return_counts=True),
                                   np.unique(so, return_counts=True))
    assert np.abs(w - wo)[both].max() <= tol
    return w, st


def test_collapsed_edge_patch():
    # triangle-like bicubic: the v=0 edge collapses to a point (singular Jacobian)
    rng = np.random.default_rng(11)
    ctrl = np.array([[(i / 3, j / 3, 0.3 * np.sin(i + 2 * j)) for j in range(4)]
                     for i in range(4)])
    ctrl[:, 0] = ctrl[0, 0]
    q = rng.uniform(-0.5, 1.5, (2000, 3))
    _edge_compare(ctrl[None], q)


def test_flat_patch_and_far_translation():
    rng = np.random.default_rng(12)
    flat = np.array([[(i / 3, j / 3, 0.0) for j in range(4)] for i in range(4)])[None]
    q = rng.uniform(-0.5, 1.5, (2000, 3))
    w, _ = _edge_compare(flat, q)
    # exact solid-angle check against the unit square formula away from it
    s1 = scenes.make(1, 2000)
    t = np.array([1234.5, -987.25, 512.0])
    _edge_compare(s1.ctrl + t, s1.queries + t, tol=1e-8)


def test_single_query_and_outside_box():
    s = scenes.make(2, 8)
    sc = G.Scene(s.ctrl)
    w, st = G.winding_numbers(sc, np.array([[0.01, 0.02, 0.03]]))
    assert st[0] == 0 and w[0] == 1.0
    far = np.array([[50.0, 0.1, 0.2], [-30.0, 40.0, 10.0], [0.0, 0.0, 99.0]])
    w, st = G.winding_numbers(sc, far)
    assert np.all(st == 0) and np.all(w == 0.0)


def test_odd_batch_sizes_equal_full_batch():
    s, sc = _scene(1)
    w, st = G.winding_numbers(sc, s.queries)
    for a, b in ((0, 1), (1, 33), (33, 161), (161, 4096)):
        wp, sp = G.winding_numbers(sc, s.queries[a:b], index_base=a)
        assert np.array_equal(wp, w[a:b]) and np.array_equal(sp, st[a:b])


@pytest.mark.parametrize("cfg", [3, 5])
def test_candidate_capacity_overflow_rerun_is_identical(cfg, monkeypatch):
    """A round whose candidate pairs overflow the capacity is discarded and re-run at
    the exact size (gwn_engine.cu, K5 publish): a scene created with a tiny initial
    estimate (GWN_PAIRS_INIT) overflows its first round and still returns the default
    scene's results bit for bit -- evals and ray reuse."""
    s = scenes.make(cfg, {3: 1 << 14, 5: 4096}[cfg])  # > 4096 candidate pairs
    sc = G.Scene(s.ctrl)
    w, st = G.winding_numbers(sc, s.queries)
    assert int(sc.stats()["candidates"]) > 4096
    monkeypatch.setenv("GWN_PAIRS_INIT", "0")
    tiny = G.Scene(s.ctrl)
    monkeypatch.delenv("GWN_PAIRS_INIT")
    w1, st1 = G.winding_numbers(tiny, s.queries)
    first = int(tiny.stats()["kernel_launches"])
    w2, st2 = G.winding_numbers(tiny, s.queries)
    second = int(tiny.stats()["kernel_launches"])
    assert np.array_equal(w1, w) and np.array_equal(st1, st)
    assert np.array_equal(w2, w) and np.array_equal(st2, st)
    assert first > second, (first, second)  # the overflowed round ran twice
    o = np.array([-0.4, 0.3, -0.2])
    d = np.array([1.0, 0.2, 0.3]) / np.linalg.norm([1.0, 0.2, 0.3])
    ts = np.linspace(0.0, 2.5, 64)
    monkeypatch.setenv("GWN_PAIRS_INIT", "0")
    tiny_r = G.Scene(s.ctrl)
    monkeypatch.delenv("GWN_PAIRS_INIT")
    wr = np.asarray(G.winding_numbers_along_ray(tiny_r, G.Ray(o, d), ts))
    wr0 = np.asarray(G.winding_numbers_along_ray(sc, G.Ray(o, d), ts))
    assert np.array_equal(wr, wr0)


def test_samples_per_edge_parity():
    s = scenes.make(1, 1000)
    for S in (2, 50, 1900):
        _edge_compare(s.ctrl, s.queries, samples_per_edge=S)


def test_concurrent_evals_on_distinct_streams():
    """gwn_eval is reentrant on distinct streams (include/gwn_b200.h): two host
    threads on one scene, including a re-shoot round built concurrently."""
    import threading
    s, sc = _scene(3)
    ref_w, ref_st = G.winding_numbers(sc, s.queries)
    out = {}

    def run(k):
        st = torch.cuda.Stream()
        q = torch.from_numpy(s.queries).cuda()
        with torch.cuda.stream(st):
            for _ in range(3):
                w, t = G.winding_numbers(sc, q)
            st.synchronize()
            out[k] = (w.cpu().numpy(), t.cpu().numpy())

    th = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for k in range(2):
        assert np.array_equal(out[k][0], ref_w) and np.array_equal(out[k][1], ref_st)


_NEWTON_PATH_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2408_04466_b200 as G
from paper_2408_04466_b200 import scenes
s = scenes.make(int(sys.argv[2]), int(sys.argv[4]) if len(sys.argv) > 4 else 1 << 15)
sc = G.Scene(s.ctrl)
w, st = G.winding_numbers(sc, torch.from_numpy(s.queries).cuda())
np.save(sys.argv[3], np.stack([w.cpu().numpy(), st.cpu().numpy().astype(np.float64)]))
"""


@pytest.mark.parametrize("cfg", [2, 3])
def test_programmatic_launch_equals_two_streams(tmp_path, cfg):
    """GWN_PDL=0 runs the fallback on a side stream joined by an event instead of
    the programmatic dependent launches; the results must be bit-identical."""
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode in ("1", "0"):
        f = str(tmp_path / f"pdl{mode}.npy")
        env = dict(os.environ, GWN_PDL=mode)
        subprocess.run([sys.executable, "-c", _NEWTON_PATH_SCRIPT, repo, str(cfg), f],
                       env=env, check=True, timeout=300)
        out[mode] = np.load(f)
    assert np.array_equal(out["1"], out["0"])


@pytest.mark.parametrize("cfg", [1, 3])
def test_newton_shared_table_equals_register_path(tmp_path, cfg):
    """Scenes of <= 96 patches run K3 Newton from the shared-memory patch
    table; GWN_NEWTON_SMEM=0 forces the register path.  Same arithmetic in the
    same order, so the results must be bit-identical."""
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode in ("1", "0"):
        f = str(tmp_path / f"r{mode}.npy")
        env = dict(os.environ, GWN_NEWTON_SMEM=mode)
        subprocess.run([sys.executable, "-c", _NEWTON_PATH_SCRIPT, repo, str(cfg), f],
                       env=env, check=True, timeout=300)
        out[mode] = np.load(f)
    assert np.array_equal(out["1"], out["0"])


@pytest.mark.parametrize("cfg", [4, 5])
def test_newton_patch_order_equals_queue_order(tmp_path, cfg):
    """Scenes beyond the shared-memory table run K3 Newton in patch order
    (per-patch item bins, k3_newton_binned) in rounds of >= 2^16 queries;
    GWN_NEWTON_BIN=0 keeps the queue order (k3_newton<false>).  The per-item
    arithmetic is the same and chi / flags are integer sums, so the results
    must be bit-identical (the small re-shoot rounds take the unbinned pass in
    both runs)."""
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for mode in ("1", "0"):
        f = str(tmp_path / f"bin{mode}.npy")
        env = dict(os.environ, GWN_NEWTON_BIN=mode)
        subprocess.run([sys.executable, "-c", _NEWTON_PATH_SCRIPT, repo, str(cfg), f, str(1 << 18)],
                       env=env, check=True, timeout=600)
        out[mode] = np.load(f)
    assert np.array_equal(out["1"], out["0"])
    assert (out["1"][1] == 0).mean() > 0.99


def _silhouette_points(ctrl, d, n_per_patch=8):
    """Surface points where the round-0 direction is tangent (n . d = 0),
    by bisection along v = const lines of each patch."""
    pts = []
    for c in ctrl:
        p = G.BicubicPatch(c)
        for v in np.linspace(0.1, 0.9, n_per_patch):
            def f(u):
                fu, fv = p.partials(u, v)
                n = np.cross(fu, fv)
                return float(n @ d) / np.linalg.norm(n)
            us = np.linspace(0.02, 0.98, 49)
            fs = [f(u) for u in us]
            for a, b, fa, fb in zip(us, us[1:], fs, fs[1:]):
                if fa * fb < 0:
                    for _ in range(80):
                        m = 0.5 * (a + b)
                        if f(m) * fa > 0:
                            a, fa = m, f(m)
                        else:
                            b = m
                    pts.append(p.point(0.5 * (a + b), v))
                    break
    return np.array(pts)


def test_forced_reshoots_and_jitters_match_oracle():
    """Queries built to trip every retry path of round 0:
    rays through a shared patch edge (grazing), rays tangent to the surface
    at a silhouette point (tangency), queries on the surface (jitter).  GPU
    statuses and w follow the oracle query by query; every grazing ray is
    re-shot on both sides."""
    s = scenes.make(2, 8)
    ctrl = s.ctrl
    d0 = O.direction(O.params().dir_seed, 0)
    rng = np.random.default_rng(11)
    edge = np.array([G.BicubicPatch(c).point(u, 0.0) for c in ctrl
                     for u in rng.uniform(0.1, 0.9, 6)])
    tang = _silhouette_points(ctrl, d0)
    onsurf = np.array([G.BicubicPatch(c).point(*rng.uniform(0.1, 0.9, 2)) for c in ctrl])
    assert len(tang) >= 4
    q = np.concatenate([edge - 0.7 * d0, tang - 0.7 * d0, onsurf])
    sc = G.Scene(ctrl)
    w, st = G.winding_numbers(sc, q)
    stats = sc.stats()
    wo, so, chi, rounds = O.scene_eval(ctrl, q)
    ne, nt = len(edge), len(tang)
    assert np.array_equal(st, so), (st, so)
    ok = st == 0
    assert np.array_equal(w[ok], wo[ok])
    assert stats["retried"] >= ne                    # every grazing ray re-shot
    assert np.all(rounds[:ne] >= 2)                  # by the oracle too
    # tangent contacts on this convex surface: re-shot or resolved as a
    # double root, the same way on both sides (statuses and w compared above)
    assert np.all(st[ne + nt:] == 1)                 # on the surface: jittered, status 1
    assert np.all(np.isin(w[ok], (0.0, 1.0)))


def test_all_hits_more_than_eight_roots():
    """A patch the z-axis crosses 9 times: x(u,v) = f(u), y(u,v) = g(v) with
    three roots each (Bernstein coefficients of the cubics), z increasing in
    u and v; the reference solver has no cap (surfaces.py:634-701)."""
    def bern_coeffs(roots, scale):
        # power coefficients of scale * prod(u - r), then to the Bernstein basis
        c = np.poly(roots)[::-1] * scale            # c0 + c1 u + c2 u^2 + c3 u^3
        return np.array([c[0], c[0] + c[1] / 3, c[0] + 2 * c[1] / 3 + c[2] / 3,
                         c[0] + c[1] + c[2] + c[3]])
    a = bern_coeffs([0.2, 0.5, 0.8], 4.0)
    b = bern_coeffs([0.15, 0.45, 0.85], 4.0)
    ctrl = np.zeros((4, 4, 3))
    for i in range(4):
        for j in range(4):
            ctrl[i, j] = (a[i], b[j], 1.0 + i / 3 + 2.7 * j / 3)
    p = G.BicubicPatch(ctrl)
    ray = G.Ray(np.array([0.0, 0.0, -1.0]), np.array([0.0, 0.0, 1.0]))
    hits = p.all_hits(ray)
    oh = O.patch_all_hits(ctrl, ray.origin, ray.direction)
    assert len(hits) == 9 and len(oh) == 9
    for h, o in zip(hits, oh):
        assert abs(h.t - o.t) < 1e-9 and h.sign == o.sign
    expect = sorted(2.0 + u + 2.7 * v for u in (0.2, 0.5, 0.8) for v in (0.15, 0.45, 0.85))
    assert np.allclose([h.t for h in hits], expect, atol=1e-9)
    # a t window inside the root set, applied on the device before the cap
    mid = p.all_hits(ray, t_window=(3.0, 4.0))
    assert [h.t for h in mid] == [h.t for h in hits if 3.0 <= h.t <= 4.0]


@pytest.mark.parametrize("cfg", [3, 5])
def test_scene_sums_match_reference_fixture(golden_dir, cfg):
    """Round-0 values against the reference's own per-patch terms summed over
    the scene (tests/golden/scene{3,5}.npz): net-boundary cancellation, the
    far field and its local expansions against per-patch reference sums."""
    g = np.load(os.path.join(golden_dir, f"scene{cfg}.npz"))
    s = scenes.make(cfg, len(g["queries"]))
    assert np.array_equal(s.queries[:len(g["queries"])], g["queries"])
    chi, bt, fl = O.scene_eval_dir(s.ctrl, g["queries"], g["d"])
    w, st = G.winding_numbers(G.Scene(s.ctrl), g["queries"])
    m = (fl == 0) & (st == 0)    # not re-shot: the round-0 direction d
    assert m.sum() >= len(m) - 2
    assert np.abs(w - g["w"])[m].max() <= W_TOL


def test_round_cache_cap_is_bit_identical():
    """Re-shoot rounds past the scene's cache (cached_rounds) are built per
    eval and freed: same results, and the scene keeps only the cached ones."""
    s = scenes.make(3, 1 << 14)
    a = G.Scene(s.ctrl)
    b = G.Scene(s.ctrl, cached_rounds=1)
    wa, sa = G.winding_numbers(a, s.queries)
    wb, sb = G.winding_numbers(b, s.queries)
    assert np.array_equal(wa, wb) and np.array_equal(sa, sb)
    ta, tb = a.stats(), b.stats()
    assert ta["rounds"] == tb["rounds"] and ta["rounds"] >= 2   # re-shoot rounds ran
    assert tb["rounds_built"] == 1 and ta["rounds_built"] >= 2
