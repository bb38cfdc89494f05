"""GPU: the reference package itself, with the INTEGRATION.md §2(a) binding
applied, running on libgwn_b200.so.

The test copies the installed reference (baseline/_ref/gwn, the unmodified
package) to a scratch directory, appends the binding exactly as
INTEGRATION.md prints it to gwn/_kernels.py (the original single_loop_batch
kept as the fallthrough), and then
  * calls gwn._kernels.single_loop_batch: results equal this package's GPU
    mirror (bit for bit) and the fan oracle;
  * runs a reference-style per-patch loop over a closed scene: chi from the
    patches' all_hits (SPEC engine CS1 step 4) and each patch's boundary term
    through the bound single_loop_batch on gwn.surfaces.patch_boundary loops
    (surfaces.py:611-626), summed over patches, against
    winding_numbers.
Skipped when baseline/_ref is not installed."""

import importlib
import os
import re
import shutil
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(REPO, "baseline", "_ref", "gwn")

import paper_2408_04466_b200 as G  # noqa: E402
from paper_2408_04466_b200 import _kernels, _lib, scenes  # noqa: E402
from oracle import oracle as O  # noqa: E402


@pytest.fixture(scope="module")
def bound_gwn(tmp_path_factory):
    if not os.path.isdir(REF):
        pytest.skip("reference not installed in baseline/_ref")
    doc = open(os.path.join(REPO, "INTEGRATION.md")).read()
    snippet = re.search(r"```python\n(# gwn/_kernels.py \(reference side\).*?)```", doc, re.S).group(1)
    # the snippet's last lines stand for "the unchanged reference code": fall
    # through to the original function instead
    head = snippet.split("    if not numba_enabled():")[0]
    binding = head.replace("def single_loop_batch(", "def single_loop_batch(") + \
        "    return _single_loop_batch_reference(loop_pts, origin, direction, hit_ts, hit_signs,\n" \
        "                                        query_ts, on_tol, t_eps)\n"
    root = tmp_path_factory.mktemp("refbound")
    pkg = root / "gwn"
    shutil.copytree(REF, pkg, ignore=shutil.ignore_patterns("__pycache__"))
    kp = pkg / "_kernels.py"
    src = kp.read_text()
    assert "def single_loop_batch(" in src
    src = src.replace("def single_loop_batch(", "def _single_loop_batch_reference(", 1)
    kp.write_text(src + "\n\n" + binding)
    os.environ["GWN_B200_LIB"] = _lib.LIB_PATH if hasattr(_lib, "LIB_PATH") else \
        os.path.join(REPO, "paper_2408_04466_b200", "libgwn_b200.so")
    saved = {k: v for k, v in sys.modules.items() if k == "gwn" or k.startswith("gwn.")}
    for k in saved:
        del sys.modules[k]
    sys.path.insert(0, str(root))
    try:
        K = importlib.import_module("gwn._kernels")
        SU = importlib.import_module("gwn.surfaces")
        assert K._gwn_b200() is not None
        yield K, SU
    finally:
        sys.path.remove(str(root))
        for k in [k for k in sys.modules if k == "gwn" or k.startswith("gwn.")]:
            del sys.modules[k]
        sys.modules.update(saved)


def test_reference_single_loop_batch_runs_on_the_gpu(bound_gwn):
    K, SU = bound_gwn
    s = scenes.make(1, 64)
    patch = G.BicubicPatch(s.ctrl[0])
    loop = SU.patch_boundary(patch, 200).points          # the reference's own sampler
    d = O.direction(O.params().dir_seed, 0)
    for p in s.queries[:16]:
        hits = patch.all_hits(G.Ray(p, d))
        ht = np.array([h.t for h in hits])
        hs = np.array([h.sign for h in hits], np.int64)
        qt = np.array([0.0, 0.1, 0.25])
        w, ok = K.single_loop_batch(loop, p, d, ht, hs, qt, 1e-9, 1e-12)
        w2, ok2 = _kernels.single_loop_batch(loop, p, d, ht, hs, qt, 1e-9, 1e-12)
        assert np.array_equal(w, w2) and np.array_equal(ok, ok2)
        if ok[0]:
            assert abs(w[0] - (hs.sum() + O.loop_fan(loop, p, d))) < 1e-12


def test_reference_style_patch_loop_equals_winding_numbers(bound_gwn):
    K, SU = bound_gwn
    s = scenes.make(3, 128)                 # 64 open patches: every boundary term matters
    patches = [G.BicubicPatch(c) for c in s.ctrl]
    loops = [SU.patch_boundary(p, 200).points for p in patches]
    d = O.direction(O.params().dir_seed, 0)
    q = s.queries[:24]
    chi, bt, fl = O.scene_eval_dir(s.ctrl, q, d)
    w_eng, st = G.winding_numbers(G.Scene(s.ctrl), q)
    for i, p in enumerate(q):
        if fl[i] or st[i]:
            continue
        w = 0.0
        for patch, loop in zip(patches, loops):
            hits = patch.all_hits(G.Ray(p, d))
            ht = np.array([h.t for h in hits])
            hs = np.array([h.sign for h in hits], np.int64)
            wk, ok = K.single_loop_batch(loop, p, d, ht, hs, np.zeros(1), 1e-9, 1e-12)
            assert ok[0] == 1
            w += wk[0]
        assert abs(w - w_eng[i]) < 1e-9, (i, w, w_eng[i])
