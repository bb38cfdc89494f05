"""Benchmark: batched generalized winding numbers on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference]

One step = one pass of the hot path (cull -> intersect -> boundary ->
reduce/re-shoot, plus the all-gather for N>1) over the rank's shard of the
config's synthetic queries.  Default workload: config 5 (BASELINE.json
configs[4], the north-star job): 15,876 bicubic patches (256 deformed closed
surfaces, 5% holes, 2% flipped duplicates), 2^26 queries, fp64 -- the largest
configuration, and it fits one B200.  Its queries are split over the N GPUs
(strong scaling: the job is fixed).

``--gpus N`` without torchrun re-launches this script under
``torch.distributed.run`` with N ranks (one per GPU, NCCL, NCCL_DEBUG=INFO).

Printed JSON (rank 0, one line):
  value      queries/s over all ranks, queries resident in HBM, device-timed
             (CUDA events, max over ranks), L2 flushed between steps
  e2e        the same metric through the public API from pinned host memory
             (H2D of the step's queries and D2H of w + status inside the timed
             region)
  roofline   the dominant kernel of the step (the exact near-field boundary
             kernel at config 5): algorithmic FP64 flops per launch (device
             counters x per-unit flops) / its CUDA-event time, vs
             the FP64 DFMA peak measured live on this GPU; `rooflines` has every
             FP64 kernel of the step
  parity     the oracle (oracle/, CPU) on the first 8,192 queries, compared
             with the GPU's results in the same run
  cpu_baseline  that oracle run's rate (the reference algorithm restated in C,
             all host threads), rank 0 at N=1; `as_shipped_reference` times
             the reference package itself (baseline/_ref) per BASELINE.md §2
"""

from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

# Algorithmic FP64 flops per unit of work (FMA = 2), DESIGN.md §4.
FLOP_NEWTON = 220.0    # K3 Newton iteration (220 per N_newton)
FLOP_ROOT = 200.0      # K3 accepted root (200 per N_root)
FLOP_SEGMENT = 31.0    # K4 exact, per (query, net segment) in the ray frame: vertex (3 sub,
                       # |r|^2 5, sqrt seed + Halley 8, u_z 1) + num 3, den 5, complex product 6
                       # (34 until the unnormalised factors of round 2 dropped 3 per vertex)
FLOP_TERM = 10.0       # K4 far field, per multipole term (Clenshaw, gwn_boundary.cu):
                       # b = D + alpha b1 + beta b2 on a complex b (4 FMA) + beta (1 FMA)
L2P_TERMS = 325        # terms of one order-24 local expansion (j <= 24, 0 <= k <= j)
FLOP_L2P = 12.0        # per local-expansion term: complex recurrence 8 + multiply-add 4

CONFIG_DESC = {
    1: "config1: single open bicubic patch, 4096 queries U[-0.5,1.5]^3",
    2: "config2: closed 6-patch bicubic cube-sphere, 2^20 queries U[-1.5,1.5]^3",
    3: "config3: open 8x8 height-field sheet (64 patches), 2^22 queries (10% within 1e-3)",
    4: "config4: 16 overlapping closed surfaces (1024 patches), 2^24 queries U[-3,3]^3",
    5: "config5: 15876 bicubic patches (256 deformed closed surfaces, 5% holes, 2% flipped "
       "duplicates), 2^26 queries uniform in the scene box",
}
PARITY_Q = 8192        # oracle parity sample (first queries of the config)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--queries", type=int, default=0,
                    help="override the job's query count (strong) / per-GPU count (weak)")
    ap.add_argument("--scaling", default=None, choices=["weak", "strong"],
                    help="strong (default for config 5): the config's queries are split over "
                         "the GPUs; weak: every GPU evaluates the config's query count")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the side measurements (other configs, far field, ray reuse, "
                         "as-shipped reference)")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    a = ap.parse_args()
    if a.scaling is None:
        a.scaling = "strong" if a.config == 5 else "weak"
    return a


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_spawn(args) -> int:
    """--gpus N > 1 outside torchrun: re-launch this script with N ranks (the
    exact code path the driver's torchrun launch runs)."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def mark(self):
        return len(self.lines)

    def stop(self, since: int = 0) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = [l.split(", ") for l in self.lines[since:] if l.count(",") >= 5] or \
            [l.split(", ") for l in self.lines if l.count(",") >= 5]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for n, v in zip(names, r[2:6]):
                if v.strip().lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(rows[0][1]),
                "reasons": sorted(reasons), "samples": len(rows)}


def _traffic(key: str):
    """DRAM bytes per launch of a kernel from the committed ncu --set full
    captures (profiles/roofline_traffic.json; same config and chunk size as
    the bench's launches), or None."""
    try:
        with open(os.path.join(HERE, "profiles", "roofline_traffic.json")) as f:
            t = json.load(f)
    except (OSError, ValueError):
        return None
    v = t.get(key)
    return v if isinstance(v, (int, float)) else None


def oracle_parity(spec, w_gpu, st_gpu, n: int, cores: int) -> tuple[dict, dict]:
    """The CPU oracle (the reference algorithm restated in C, oracle/) on the
    first n queries with all host threads: parity against the GPU's results
    of the same run, and the cpu_baseline rate."""
    from oracle import oracle as O
    q = spec.queries[:n]
    O.scene_eval(spec.ctrl, q[:16], qidx=np.arange(16), nthreads=cores)  # warm
    t = time.perf_counter()
    wo, so, _, _ = O.scene_eval(spec.ctrl, q, qidx=np.arange(n), nthreads=cores)
    dt = time.perf_counter() - t
    wg, sg = w_gpu[:n], st_gpu[:n]
    both = (sg == 0) & (so == 0)
    d = np.abs(wg - wo)[both]
    cls_g, cls_o = np.round(wg[both]), np.round(wo[both])
    far = np.abs(wo[both] - np.round(wo[both])) > 1e-6
    par = {"queries": n, "both_status_ok": int(both.sum()),
           "status_equal": int((sg == so).sum()),
           "max_abs_dw": float(d.max()) if d.size else 0.0,
           "rms_dw": float(np.sqrt(np.mean(d * d))) if d.size else 0.0,
           "rounded_w_equal": int((cls_g == cls_o).sum()),
           "non_integer_w": int(far.sum()),
           "tolerance": "north star: |dw| <= 1e-6; integer classification exact",
           "pass": bool(d.size and d.max() <= 1e-6 and both.mean() > 0.99)}
    base = {"value": n / dt, "unit": "queries/s", "cores": cores, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": f"first {n} queries of {CONFIG_DESC[spec.config].split(':')[0]} "
                      f"({dt:.1f} s; oracle/gwn_oracle.c, the reference algorithm restated in C "
                      f"with subdivided seeding, exact boundary sum, {cores} threads)"}
    return par, base


def run_reference(args, spec, rank, world):
    """--impl reference: the CPU oracle port on the host cores (rank 0 only),
    each step a bounded sample of the workload."""
    if rank != 0:
        return 0
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    n = 256
    while True:  # bounded per-step sample: >= ~4 s of CPU work per step
        t = time.perf_counter()
        O.scene_eval(spec.ctrl, spec.queries[:n], qidx=np.arange(n), nthreads=cores)
        dt = time.perf_counter() - t
        if dt > 4.0 or n >= len(spec.queries):
            break
        n = min(len(spec.queries), n * 2)
    for _ in range(args.warmup):
        O.scene_eval(spec.ctrl, spec.queries[:n], qidx=np.arange(n), nthreads=cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.scene_eval(spec.ctrl, spec.queries[:n], qidx=np.arange(n), nthreads=cores)
    el = time.perf_counter() - t0
    v = n * args.steps / el
    line = {
        "impl": "reference", "metric": "winding-number queries/sec", "value": v,
        "unit": "queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY.md §8(d))",
        "config": {"workload": CONFIG_DESC[spec.config], "n_patches": spec.n_patches,
                   "queries": int(len(spec.queries)), "sample_per_step": n},
        "cpu_baseline": {"value": v, "unit": "queries/s", "cores": cores, "kind": "port",
                         "cpu_model": cpu_model(),
                         "sample": f"first {n} queries per step, oracle/gwn_oracle.c (the "
                                   "reference algorithm restated in C; the reference itself is "
                                   "Python with no bicubic type or engine, DESIGN.md §8)"},
        "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def side_config(G, torch, cfg: int, dev, stream, k: int = 5) -> dict:
    """Another BASELINE config on one GPU, device-resident, L2 flushed: the
    config's full query count, best-effort per-stage split (extra key)."""
    from paper_2408_04466_b200 import scenes
    s = scenes.make(cfg)
    sc = G.Scene(s.ctrl, device=dev.index)
    q = torch.from_numpy(s.queries).to(dev)
    w = torch.empty(len(q), dtype=torch.float64, device=dev)
    st = torch.empty(len(q), dtype=torch.int8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):
        G.winding_numbers(sc, q, out=(w, st), stream=stream.cuda_stream)
    torch.cuda.synchronize()
    ms = 0.0
    for _ in range(k):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        G.winding_numbers(sc, q, out=(w, st), stream=stream.cuda_stream)
        b.record(stream)
        torch.cuda.synchronize()
        ms += a.elapsed_time(b)
    return {"workload": CONFIG_DESC[cfg], "queries": len(q), "n_patches": s.n_patches,
            "value": len(q) / (ms / k * 1e-3), "unit": "queries/s", "ms_per_step": ms / k,
            "steps": k, "warmup": 3}


def far_field_side(G, torch, dev, stream, nq=1 << 18, k=2) -> dict:
    """config 5's boundary term with the far field against
    the exact fan sum (GWN_FARFIELD=0), both device-timed, and the largest
    |dw| between the two."""
    from paper_2408_04466_b200 import scenes
    s = scenes.make(5, nq)
    q = torch.from_numpy(s.queries).to(dev)
    res = {}
    for mode in ("exact", "far"):
        old = os.environ.get("GWN_FARFIELD")
        if mode == "exact":
            os.environ["GWN_FARFIELD"] = "0"
        try:
            sc = G.Scene(s.ctrl, device=dev.index)   # the switch is read at scene creation
        finally:
            if mode == "exact":
                if old is None:
                    os.environ.pop("GWN_FARFIELD", None)
                else:
                    os.environ["GWN_FARFIELD"] = old
        G.winding_numbers(sc, q, stream=stream.cuda_stream)
        sc.set_timing(True)
        best, stt, w, st = float("inf"), None, None, None
        for _ in range(k):
            w, st = G.winding_numbers(sc, q, stream=stream.cuda_stream)
            t = sc.stats()
            if t["ms_boundary"] < best:
                best, stt = t["ms_boundary"], t
        sc.set_timing(False)
        res[mode] = (best, w.cpu().numpy(), st.cpu().numpy(), stt)
    ok = (res["exact"][2] == 0) & (res["far"][2] == 0)
    return {"workload": f"config5 scene, {nq} queries, boundary term (K4)",
            "ms_exact": res["exact"][0], "ms_far_field": res["far"][0],
            "speedup": res["exact"][0] / res["far"][0],
            "far_pairs": res["far"][3]["far_pairs"], "near_pairs": res["far"][3]["near_pairs"],
            "exact_segment_pairs": res["far"][3]["boundary_segments"],
            "exact_segment_pairs_without": res["exact"][3]["boundary_segments"],
            "max_abs_dw": float(np.abs(res["exact"][1] - res["far"][1])[ok].max()),
            "status_equal": bool(np.array_equal(res["exact"][2], res["far"][2]))}


def ray_reuse_side(G, torch, cfg, dev, stream, n=256, k=3) -> dict:
    """voxel centres of a config's scene box at n^3 through
    gwn_eval_rays (n^2 rays along +x) against gwn_eval of the same points,
    both device-resident, CUDA events on `stream`."""
    from paper_2408_04466_b200 import scenes
    s = scenes.make(cfg, 8)
    sc = G.Scene(s.ctrl, device=dev.index)
    bb = sc.aabb()
    lo, hi = bb.min_corner, bb.max_corner
    c = (torch.arange(n, dtype=torch.float64, device=dev) + 0.5) / n
    ax = [float(lo[i]) + c * float(hi[i] - lo[i]) for i in range(3)]
    Y, Z = torch.meshgrid(ax[1], ax[2], indexing="ij")
    org = torch.stack([torch.full_like(Y, float(lo[0])), Y, Z], -1).reshape(-1, 3)
    ts = (c * float(hi[0] - lo[0])).repeat(n * n)
    offs = torch.arange(n * n + 1, dtype=torch.int64, device=dev) * n
    pts = org.repeat_interleave(n, 0)
    pts[:, 0] += ts
    w_pp = torch.empty(n ** 3, dtype=torch.float64, device=dev)
    st_pp = torch.empty(n ** 3, dtype=torch.int8, device=dev)

    def t_of(fn):
        fn()
        torch.cuda.synchronize()
        best = float("inf")
        for _ in range(k):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        return best

    res = {}
    ms_r = t_of(lambda: res.update(r=G.winding_numbers_rays(
        sc, org, [1.0, 0.0, 0.0], ts, offs, stream=stream.cuda_stream, check=False)))
    ms_p = t_of(lambda: G.winding_numbers(sc, pts, out=(w_pp, st_pp), stream=stream.cuda_stream))
    w_r, st_r = res["r"]
    ok = (st_r == 0) & (st_pp == 0)
    diff = float((w_r - w_pp).abs()[ok].max()) if bool(ok.any()) else 0.0
    return {"workload": f"config{cfg} scene box voxelized at {n}^3 = {n ** 3} voxel centres, "
                        f"{n * n} rays along +x (SPEC.md:398-407)",
            "value": n ** 3 / (ms_r * 1e-3), "unit": "points/s", "ms": ms_r,
            "rays_cast": sc.rays_cast, "per_point_value": n ** 3 / (ms_p * 1e-3),
            "per_point_ms": ms_p, "speedup": ms_p / ms_r, "max_abs_diff_vs_per_point": diff}


def rooflines(stt: dict, peak_tf: float, ms_step: float, config: int) -> dict:
    """Every FP64 kernel of the step: algorithmic flops (device counters x
    per-unit flops) / its event-timed duration, against the live DFMA peak."""
    ks = {
        "k_ff_near (K4 exact near field)": (
            stt.get("ms_k4_exact", 0.0), stt["boundary_segments"] * FLOP_SEGMENT,
            f"{int(stt['boundary_segments'])} (query, segment) pairs x {FLOP_SEGMENT:.0f} flop",
            "k_ff_near"),
        "k_ff_fill + k_ff_far_eval (K4 far field)": (
            stt.get("ms_k4_far", 0.0),
            stt.get("far_terms", 0) * FLOP_TERM + stt.get("local_evals", 0) * L2P_TERMS * FLOP_L2P,
            f"{int(stt.get('far_terms', 0))} multipole terms x {FLOP_TERM:.0f} flop "
            f"({int(stt['far_pairs'])} per-pair far (query, cycle) expansions) + "
            f"{int(stt.get('local_evals', 0))} local expansions x {L2P_TERMS} terms x "
            f"{FLOP_L2P:.0f} flop", "k_ff_fill"),
        "k3_newton_binned (K3 Newton + record)"
        if config == 5 or config == 4 else "k3_newton (K3 Newton + record)": (
            stt["ms_k3_newton"], stt["newton_iters"] * FLOP_NEWTON + stt["roots"] * FLOP_ROOT,
            f"{int(stt['newton_iters'])} iterations x {FLOP_NEWTON:.0f} + {int(stt['roots'])} "
            f"roots x {FLOP_ROOT:.0f} flop", "k3_newton"),
    }
    if stt.get("ms_k4_exact", 0.0) <= 0.0 and stt["ms_boundary"] > 0:
        ks["k_boundary_e (K4 exact)"] = (stt["ms_boundary"],
                                         stt["boundary_segments"] * FLOP_SEGMENT,
                                         "all (query, segment) pairs", "k_boundary_e")
    out = {}
    for name, (ms, flops, units, key) in ks.items():
        if ms <= 0.0 or flops <= 0.0:
            continue
        ach = flops / (ms * 1e-3) / 1e12
        out[name] = {"bound": "fp64", "achieved": ach, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": ach / peak_tf if peak_tf else None,
                     "traffic": _traffic(f"c{config}:{key}"),
                     "kernel_ms_per_step": ms, "kernel_share_of_step": ms / ms_step,
                     "algorithmic_units": units,
                     "peak_source": "FP64 DFMA-chain microbenchmark run live on this GPU "
                                    "(MEASURED_PEAKS.json has no FP64 entry)"}
    return out


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_spawn(args)
    # test hook: GWN_BENCH_ONE_GPU=1 runs every rank on cuda:0 over gloo, so
    # the N > 1 code path (sharding, packed all-gather, max over ranks) can be
    # exercised on a one-GPU box; never used for reported numbers
    one_gpu = os.environ.get("GWN_BENCH_ONE_GPU") == "1"
    if world != args.gpus:
        raise SystemExit(f"WORLD_SIZE={world} but --gpus {args.gpus}")
    if one_gpu:
        local = 0
    from paper_2408_04466_b200 import scenes
    base = args.queries or scenes.FULL_QUERIES[args.config]
    total = base * world if args.scaling == "weak" else base
    spec = scenes.make(args.config, total)
    if args.impl == "reference":
        return run_reference(args, spec, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2408_04466_b200 as G

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    n_total = len(spec.queries)
    from paper_2408_04466_b200.distributed import gather_packed, packed_shard, shard_bounds
    s0, s1, per = shard_bounds(n_total, rank, world)
    local_q = np.ascontiguousarray(spec.queries[s0:s1])
    nq = len(local_q)
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()
    t = time.perf_counter()
    sc = G.Scene(spec.ctrl, device=local)
    torch.cuda.synchronize()
    scene_build_s = time.perf_counter() - t
    q_dev = torch.from_numpy(local_q).to(dev)
    w_dev = torch.empty(nq, dtype=torch.float64, device=dev)
    st_dev = torch.empty(nq, dtype=torch.int8, device=dev)
    q_pin = torch.from_numpy(local_q).pin_memory()
    w_pin = torch.empty(nq, dtype=torch.float64).pin_memory()
    st_pin = torch.empty(nq, dtype=torch.int8).pin_memory()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    # N > 1: the engine writes into this rank's packed (w, status) block and
    # ONE all-gather assembles every rank's results (distributed.py)
    pbuf, w_pk, st_pk = packed_shard(per, dev)
    g_all = torch.empty(world * pbuf.numel(), dtype=torch.uint8, device=dev)
    if world > 1:
        w_dev, st_dev = w_pk[:nq], st_pk[:nq]

    def step_device():
        G.winding_numbers(sc, q_dev, index_base=s0, out=(w_dev, st_dev),
                          stream=stream.cuda_stream)
        if world > 1:
            gather_packed(pbuf, world, n_total, out=g_all)

    def step_e2e():
        G.winding_numbers(sc, q_pin, index_base=s0, out=(w_pin, st_pin),
                          stream=stream.cuda_stream)
        if world > 1:
            w_pk[:nq].copy_(w_pin, non_blocking=True)
            st_pk[:nq].copy_(st_pin, non_blocking=True)
            gather_packed(pbuf, world, n_total, out=g_all)

    def timed(fn, k):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(k)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        launches = 0
        for a, b in evs:
            flush.zero_()                      # L2 flush between steps (untimed)
            a.record(stream)
            fn()
            b.record(stream)
            launches += int(sc.stats()["kernel_launches"])
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = sum(a.elapsed_time(b) for a, b in evs)
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item()), launches

    # first evaluation: builds the re-shoot rounds' structures (cached on the
    # scene) -- reported, not timed as a step
    torch.cuda.synchronize()
    t = time.perf_counter()
    step_device()
    torch.cuda.synchronize()
    first_eval_s = time.perf_counter() - t
    st0 = sc.stats()
    clocks = ClockSampler(local)
    clocks.start()
    warm = max(3, args.warmup)
    for _ in range(warm - 1):
        step_device()
    torch.cuda.synchronize()
    mark = clocks.mark()
    ms_dev, launches = timed(step_device, args.steps)
    clock_info = clocks.stop(mark)
    if one_gpu and world > 1:  # test hook: the gathered results equal one full eval
        from paper_2408_04466_b200.distributed import unpad
        torch.cuda.synchronize()
        wg, sg = unpad(*gather_packed(pbuf, world, n_total, out=g_all), per, n_total)
        if rank == 0:
            w1, s1_ = G.winding_numbers(sc, torch.from_numpy(spec.queries).to(dev))
            ok = torch.equal(wg, w1) and torch.equal(sg, s1_)
            print(f"one-gpu gather check: {'identical' if ok else 'MISMATCH'}", file=sys.stderr,
                  flush=True)
            if not ok:
                raise SystemExit("sharded + gathered results differ from one full eval")
    w_host = w_dev[:min(nq, PARITY_Q)].cpu().numpy()
    st_host = st_dev[:min(nq, PARITY_Q)].cpu().numpy()
    for _ in range(warm):   # the host path's own workspace and copy streams settle
        step_e2e()
    ms_e2e, _ = timed(step_e2e, args.steps)
    e2e_equal = bool(torch.equal(w_pin[:1024], w_dev[:1024].cpu()))

    # the e2e step's PCIe floor: the same bytes copied alone (inputs H2D and
    # (w, status) D2H on two streams at once), no compute
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    q_cp = torch.empty_like(q_dev)

    def step_copies():
        s_in.wait_stream(stream)
        s_out.wait_stream(stream)
        with torch.cuda.stream(s_in):
            q_cp.copy_(q_pin, non_blocking=True)
        with torch.cuda.stream(s_out):
            w_pin.copy_(w_dev, non_blocking=True)
            st_pin.copy_(st_dev, non_blocking=True)
        stream.wait_stream(s_in)
        stream.wait_stream(s_out)

    step_copies()
    ms_cp, _ = timed(step_copies, args.steps)

    # ---- per-kernel times and device counters of one step: the library
    # records CUDA events around each kernel on `stream` (set_timing)
    sc.set_timing(True)
    flush.zero_()
    G.winding_numbers(sc, q_dev, index_base=s0, out=(w_dev, st_dev), stream=stream.cuda_stream)
    stt = sc.stats()
    sc.set_timing(False)
    peak_tf, _ = G.fp64_peak(local)
    ms_step = ms_dev / args.steps
    rl = rooflines(stt, peak_tf, ms_step, args.config)
    head_name = max(rl, key=lambda k: rl[k]["kernel_ms_per_step"]) if rl else None

    value = n_total / (ms_step * 1e-3)
    e2e = n_total / (ms_e2e * 1e-3 / args.steps)
    out = None
    if rank == 0:
        head = dict(rl[head_name], kernel=head_name) if head_name else None
        out = {
            "metric": "winding-number queries/sec", "value": value, "unit": "queries/s",
            "n_gpus": world, "steps": args.steps, "warmup": warm,
            "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, SURVEY.md §8(d); no public dataset)",
            "config": {"workload": CONFIG_DESC[args.config], "n_patches": spec.n_patches,
                       "queries": n_total, "queries_per_gpu": per,
                       "net_boundary_segments": sc.n_net_segments,
                       "boundary_entries": sc.n_far_cycles,
                       "parallelism": f"dp{world} (queries sharded, scene replicated, "
                                      "one all-gather)",
                       "l2": "flushed between steps (256 MiB write)"},
            "nominal_pairs_per_s": value * spec.n_patches,
            "candidate_pairs_per_s": stt["candidates"] / (ms_step * 1e-3) * world,
            "e2e": {"value": e2e, "unit": "queries/s", "h2d_bytes_per_step": int(nq * 24),
                    "d2h_bytes_per_step": int(nq * 9), "results_equal_device_path": e2e_equal},
            "e2e_copy_floor": {
                "value": n_total / (ms_cp * 1e-3 / args.steps), "unit": "queries/s",
                "ms_per_step": ms_cp / args.steps, "frac": ms_cp / ms_e2e,
                "note": "the e2e step's input and output copies alone (pinned host memory, "
                        "H2D and D2H concurrently on two streams); frac = floor time / "
                        "e2e time"},
            "gpu_launches": launches,
            "roofline": head,
            "rooflines": rl,
            "scene_build_s": scene_build_s,
            "local_expansions": sc.local_expansions,
            "first_eval_s": first_eval_s,
            "rounds_built": int(st0["rounds_built"]),
            "first_eval_round_build_ms": st0["ms_round_build"],
            "one_shot_s": scene_build_s + first_eval_s,
            "stage_ms": {"cull": stt["ms_cull"],
                         # candidate test (+ the patch-bin scan and scatter of the Newton queue)
                         "k3_candidates": stt["ms_k3_candidates"],
                         "k3_fallback": stt["ms_k3_fallback"], "k3_newton": stt["ms_k3_newton"],
                         "boundary": stt["ms_boundary"], "k4_far": stt["ms_k4_far"],
                         "k4_exact": stt["ms_k4_exact"], "finalize": stt["ms_other"]},
            "counters": {k: stt[k] for k in ("candidates", "nodes", "newton_iters", "roots",
                                             "k3_newton_items", "k3_fallback_items",
                                             "boundary_segments", "far_pairs", "far_terms",
                                             "near_pairs", "retried", "rounds")},
            "clocks": clock_info,
        }
    if world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        par, base = oracle_parity(spec, w_host, st_host, min(nq, PARITY_Q), cores)
        out["parity"] = par
        out["cpu_baseline"] = base
        if not args.no_extras:
            try:
                from oracle import ref_asshipped
                out["as_shipped_reference"] = ref_asshipped.measure(cores)
            except Exception as e:  # the reference package travels in baseline/_ref
                out["as_shipped_reference"] = {"unavailable": f"{type(e).__name__}: {e}"}
    if world == 1 and not args.no_extras:
        # the side measurements build their own scenes: release the headline
        # job's scene and cached 2^26-query workspace first
        del sc, q_dev, w_dev, st_dev, flush, pbuf, w_pk, st_pk, g_all
        import gc
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        G.release_caches(local)
        extra = {}
        for cfg in (2, 3, 4):
            if cfg != args.config:
                extra[f"config{cfg}"] = side_config(G, torch, cfg, dev, stream)
        out["other_configs"] = extra
        out["far_field"] = far_field_side(G, torch, dev, stream)
        out["ray_reuse"] = ray_reuse_side(G, torch, 4, dev, stream)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
