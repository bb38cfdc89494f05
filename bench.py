"""Benchmark: batched generalized winding numbers on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl b200|reference]

One step = one pass of the hot path (cull -> intersect -> boundary ->
reduce/re-shoot, plus the all-gather for N>1) over the rank's shard of the
config's synthetic queries.  Default workload: config 2 (BASELINE.json
configs[1]): closed 6-patch bicubic surface, 2^20 queries, fp64.

Printed JSON (rank 0, one line):
  value      queries/s over all ranks, queries resident in HBM, device-timed
             (CUDA events, max over ranks), L2 flushed between steps
  e2e        the same metric through the public API from pinned host memory
             (H2D of the step's queries and D2H of w + status inside the timed
             region)
  roofline   K3 (the dominant kernel at config 2) algorithmic FP64 flops per
             launch (device counters x per-stage flop constants, DESIGN.md
             §Measurement) / its event-timed duration, vs the FP64 DFMA peak
             measured live on this GPU
  cpu_baseline  the CPU oracle port (oracle/, all host threads) on a bounded
             sample of the same workload, rank 0 at N=1
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

# Algorithmic FP64 flops per unit of work (FMA = 2).  K3: SURVEY.md §8(d)'s
# per-unit figures for the reference algorithm's work units (a Newton
# iteration evaluates the map and its partials in the Bernstein basis and
# solves the 2x2 system; an accepted root adds C, the normal and the record
# tests).  The kernel's Horner form of the same iteration executes fewer
# (142), so achieved counts work done, not instructions issued.
FLOP_NEWTON = 220.0    # K3 Newton iteration (220 per N_newton)
FLOP_ROOT = 200.0      # K3 accepted root (200 per N_root)
FLOP_SEGMENT = 34.0    # K4 per (query, net segment) in the ray frame: vertex (3 sub, |r|^2 5,
                       # rsqrt seed + Halley 8, u 4) + num 3, den 5, complex product 6

CONFIG_DESC = {
    1: "config1: single open bicubic patch, 4096 queries U[-0.5,1.5]^3",
    2: "config2: closed 6-patch bicubic cube-sphere, 2^20 queries U[-1.5,1.5]^3",
    3: "config3: open 8x8 height-field sheet (64 patches), 2^22 queries (10% within 1e-3)",
    4: "config4: 16 overlapping closed surfaces (1024 patches), 2^24 queries U[-3,3]^3",
    5: "config5: 15876 patches (256 surfaces, 5% holes, 2% flipped duplicates), 2^26 queries",
}


def _traffic(kname: str, config: int, n: int):
    """DRAM bytes per launch of the roofline kernel from the committed ncu
    --set full capture (profiles/roofline_traffic.json, config 2 at 2^20
    queries), or None for another workload."""
    if config != 2 or n != (1 << 20):
        return None
    try:
        with open(os.path.join(HERE, "profiles", "roofline_traffic.json")) as f:
            t = json.load(f)
    except (OSError, ValueError):
        return None
    return t.get(kname.split(" ")[0])


def _cull_roofline(stt, nq):
    """K2 `k_cull_grid` against HBM: algorithmic DRAM bytes = per query the
    position read (24 B), its ray-frame projection and chi / flag
    accumulators written (24 + 8 B), the cell range read (8 B); per candidate
    the (slot, leaf) pair written (8 B).  Cell entries are L2-resident."""
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            peak, src = json.load(f)["hbm_gbs"], "MEASURED_PEAKS.json hbm_gbs (copy, burst)"
    except (OSError, ValueError, KeyError):
        peak, src = 7700.0, "B200_PROFILING.md fallback"
    ms = stt["ms_cull"]
    algo = 64.0 * nq + 8.0 * stt["candidates"]
    ach = algo / (ms * 1e-3) / 1e9 if ms > 0 else 0.0
    return {"bound": "hbm", "kernel": "k_cull_grid (K2)", "achieved": ach, "peak": peak,
            "unit": "GB/s", "frac": ach / peak if peak else None,
            "traffic": _traffic("k_cull_grid", 2, nq), "algorithmic_bytes": algo,
            "kernel_ms": ms, "peak_source": src,
            "note": "latency-bound (ncu: long-scoreboard stalls on the dependent "
                    "position -> cell -> entry loads), not bandwidth-bound"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--queries", type=int, default=0,
                    help="override the per-GPU query count (weak scaling) / total (strong)")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: every GPU evaluates the config's query count (total grows "
                         "with N); strong: the config's queries are split over the GPUs")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-far-field", action="store_true",
                    help="skip the SURVEY §8(f4) far-field side measurement (config 5)")
    ap.add_argument("--no-ray-reuse", action="store_true",
                    help="skip the SURVEY §8(f1) ray-reuse side measurement")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    return ap.parse_args()


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
                 "--format=csv,noheader,nounits", "-lms", "50"],
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
        time.sleep(0.12)
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


def cpu_baseline(spec, seconds: float) -> dict:
    """Time the CPU oracle port (all host threads) on a bounded sample."""
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    n = 1024
    q = spec.queries
    O.scene_eval(spec.ctrl, q[:64])                     # warm caches / thread pool
    while True:
        t = time.perf_counter()
        O.scene_eval(spec.ctrl, q[:n], qidx=np.arange(n), nthreads=cores)
        dt = time.perf_counter() - t
        if dt >= seconds / 4 or n >= len(q):
            break
        n = min(len(q), n * 4)
    return {"value": n / dt, "unit": "queries/s", "cores": cores, "kind": "port",
            "sample": f"first {n} queries of {CONFIG_DESC[spec.config].split(':')[0]} "
                      f"({dt:.1f} s, oracle/gwn_oracle.c, {cores} threads)"}


def run_reference(args, spec, rank, world):
    """--impl reference: the CPU oracle port on the host cores (rank 0 only)."""
    if rank != 0:
        return 0
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    # bounded per-step sample: ~2 s of CPU work per step
    n = 2048
    while True:
        t = time.perf_counter()
        O.scene_eval(spec.ctrl, spec.queries[:n], qidx=np.arange(n), nthreads=cores)
        dt = time.perf_counter() - t
        if dt > 1.0 or n >= len(spec.queries):
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
                         "sample": f"first {n} queries per step, oracle/gwn_oracle.c"},
        "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def boundary_roofline(G, torch, dev, stream, peak_tf, nq=1 << 20, k=3):
    """K4's exact fan kernel (`k_boundary_e`, far field off) on config 3's scene,
    2^20 queries: algorithmic FP64 flops (device segment counter x
    FLOP_SEGMENT) over its CUDA-event time, best of k -- a side measurement:
    the bench workload (config 2) is closed and has no net boundary."""
    from paper_2408_04466_b200 import scenes
    s = scenes.make(3, nq)
    # the exact fan kernel on its own (the f4 far field would take most of
    # config 3's pairs; it has its own side measurement, `far_field`)
    old = os.environ.get("GWN_FARFIELD")
    os.environ["GWN_FARFIELD"] = "0"
    try:
        sc = G.Scene(s.ctrl)
    finally:
        if old is None:
            os.environ.pop("GWN_FARFIELD", None)
        else:
            os.environ["GWN_FARFIELD"] = old
    q = torch.from_numpy(s.queries).to(dev)
    G.winding_numbers(sc, q, stream=stream.cuda_stream)
    sc.set_timing(True)
    best, segs = float("inf"), 0
    for _ in range(k):
        G.winding_numbers(sc, q, stream=stream.cuda_stream)
        st = sc.stats()
        if st["ms_boundary"] < best:
            best, segs = st["ms_boundary"], st["boundary_segments"]
    sc.set_timing(False)
    ach = segs * FLOP_SEGMENT / (best * 1e-3) / 1e12
    return {"workload": f"config3 scene (64 patches, {sc.n_net_segments} net segments), "
                        f"{nq} queries", "kernel": "k_boundary_e (K4 fan term)",
            "bound": "fp64", "achieved": ach, "peak": peak_tf, "unit": "TFLOP/s",
            "frac": ach / peak_tf if peak_tf else None, "kernel_ms": best,
            "traffic": _traffic("k_boundary_e_config3_2^20", 2, 1 << 20) if nq == 1 << 20
            else None,
            "segment_pairs": segs}


def far_field(G, torch, dev, stream, nq=1 << 18, k=2):
    """SURVEY §8(f) f4 side measurement: config 5's boundary term (the 64M x 16K
    north-star scene, 2^18 queries here) with the far-field expansion against
    the exact fan sum -- both device-timed K4 stages, best of k, and the
    largest |dw| between the two."""
    from paper_2408_04466_b200 import scenes
    s = scenes.make(5, nq)
    q = torch.from_numpy(s.queries).to(dev)
    res = {}
    for mode in ("exact", "far"):
        old = os.environ.get("GWN_FARFIELD")
        if mode == "exact":
            os.environ["GWN_FARFIELD"] = "0"
        try:
            sc = G.Scene(s.ctrl)          # the switch is read at scene creation
        finally:
            if mode == "exact":
                if old is None:
                    os.environ.pop("GWN_FARFIELD", None)
                else:
                    os.environ["GWN_FARFIELD"] = old
        w, st = G.winding_numbers(sc, q, stream=stream.cuda_stream)
        sc.set_timing(True)
        best, stt = float("inf"), None
        for _ in range(k):
            w, st = G.winding_numbers(sc, q, stream=stream.cuda_stream)
            t = sc.stats()
            if t["ms_boundary"] < best:
                best, stt = t["ms_boundary"], t
        sc.set_timing(False)
        res[mode] = (best, w.cpu().numpy(), st.cpu().numpy(), stt, sc.n_far_cycles)
    ok = (res["exact"][2] == 0) & (res["far"][2] == 0)
    return {"workload": f"config5 scene ({s.n_patches} patches), {nq} queries, boundary term (K4)",
            "ms_exact": res["exact"][0], "ms_far_field": res["far"][0],
            "speedup": res["exact"][0] / res["far"][0],
            "far_cycles": res["far"][4], "far_pairs": res["far"][3]["far_pairs"],
            "exact_segment_pairs": res["far"][3]["boundary_segments"],
            "exact_segment_pairs_without": res["exact"][3]["boundary_segments"],
            "max_abs_dw": float(np.abs(res["exact"][1] - res["far"][1])[ok].max()),
            "status_equal": bool(np.array_equal(res["exact"][2], res["far"][2]))}


def ray_reuse(G, torch, sc, dev, stream, n=256, k=5):
    """voxel centres of the scene AABB at n^3 through
    gwn_eval_rays (n^2 rays along +x) against gwn_eval of the same points,
    both device-resident, CUDA events on `stream`."""
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
        # best of k single calls (CUDA events on `stream`), after two warm-ups
        fn()
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
            if os.environ.get("GWN_RR_DEBUG"):
                print("ray_reuse call ms", a.elapsed_time(b), file=sys.stderr, flush=True)
        return best

    res = {}
    ms_r = t_of(lambda: res.update(r=G.winding_numbers_rays(
        sc, org, [1.0, 0.0, 0.0], ts, offs, stream=stream.cuda_stream, check=False)))
    ms_p = t_of(lambda: G.winding_numbers(sc, pts, out=(w_pp, st_pp), stream=stream.cuda_stream))
    w_r, st_r = res["r"]
    ok = (st_r == 0) & (st_pp == 0)
    diff = float((w_r - w_pp).abs()[ok].max()) if bool(ok.any()) else 0.0
    return {"workload": f"voxelize scene AABB at {n}^3 = {n ** 3} voxel centres, {n * n} rays "
                        "along +x (SPEC.md:398-407)",
            "value": n ** 3 / (ms_r * 1e-3), "unit": "points/s", "ms": ms_r,
            "rays_cast": sc.rays_cast, "per_point_value": n ** 3 / (ms_p * 1e-3),
            "per_point_ms": ms_p, "speedup": ms_p / ms_r, "max_abs_diff_vs_per_point": diff}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: GWN_BENCH_ONE_GPU=1 runs every rank on cuda:0 over gloo, so
    # the N > 1 code path (sharding, packed all-gather, max over ranks) can be
    # exercised on a one-GPU box; never used for reported numbers
    one_gpu = os.environ.get("GWN_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    from paper_2408_04466_b200 import scenes
    base = args.queries or scenes.FULL_QUERIES[args.config]
    # weak scaling: N x the per-GPU count from the same seeded generator
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
    from paper_2408_04466_b200.distributed import shard_bounds
    s0, s1, per = shard_bounds(n_total, rank, world)
    local_q = np.ascontiguousarray(spec.queries[s0:s1])
    nq = len(local_q)
    sc = G.Scene(spec.ctrl, device=local)
    stream = torch.cuda.current_stream(dev)
    q_dev = torch.from_numpy(local_q).to(dev)
    w_dev = torch.empty(nq, dtype=torch.float64, device=dev)
    st_dev = torch.empty(nq, dtype=torch.int8, device=dev)
    q_pin = torch.from_numpy(local_q).pin_memory()
    w_pin = torch.empty(nq, dtype=torch.float64).pin_memory()
    st_pin = torch.empty(nq, dtype=torch.int8).pin_memory()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    # N > 1: the engine writes into this rank's packed (w, status) block and
    # ONE all-gather assembles every rank's results (distributed.py)
    from paper_2408_04466_b200.distributed import gather_packed, packed_shard
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

    clocks = ClockSampler(local)
    clocks.start()
    for _ in range(max(3, args.warmup)):
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
            w1, s1 = G.winding_numbers(sc, torch.from_numpy(spec.queries).to(dev))
            ok = torch.equal(wg, w1) and torch.equal(sg, s1)
            print(f"one-gpu gather check: {'identical' if ok else 'MISMATCH'}", file=sys.stderr,
                  flush=True)
            if not ok:
                raise SystemExit("sharded + gathered results differ from one full eval")
    for _ in range(2):
        step_e2e()
    ms_e2e, _ = timed(step_e2e, args.steps)

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

    for _ in range(2):
        step_copies()
    ms_cp, _ = timed(step_copies, args.steps)

    # ---- roofline of the dominant FP64 kernel, measured live: the library
    # records CUDA events around each kernel on `stream` (set_timing)
    sc.set_timing(True)
    kk = 3
    agg = {}
    for _ in range(kk):
        flush.zero_()
        G.winding_numbers(sc, q_dev, index_base=s0, out=(w_dev, st_dev),
                          stream=stream.cuda_stream)
        for k, v in sc.stats().items():
            agg[k] = agg.get(k, 0) + v
    sc.set_timing(False)
    stt = {k: v / kk for k, v in agg.items()}
    peak_tf, _ = G.fp64_peak(local)
    kernels = {
        "k3_newton (K3 Newton + record)": (stt["ms_k3_newton"],
                                           stt["newton_iters"] * FLOP_NEWTON
                                           + stt["roots"] * FLOP_ROOT),
        "k_boundary (K4 fan term)": (stt["ms_boundary"], stt["boundary_segments"] * FLOP_SEGMENT),
    }
    kname, (kms, kflops) = max(kernels.items(), key=lambda kv: kv[1][0])
    achieved = kflops / (kms * 1e-3) / 1e12 if kms > 0 else 0.0

    value = n_total / (ms_dev * 1e-3 / args.steps)
    e2e = n_total / (ms_e2e * 1e-3 / args.steps)
    out = None
    if rank == 0:
        out = {
            "metric": "winding-number queries/sec", "value": value, "unit": "queries/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup),
            "ms_per_step": ms_dev / args.steps, "higher_is_better": True,
            "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, SURVEY.md §8(d); no public dataset)",
            "config": {"workload": CONFIG_DESC[args.config], "n_patches": spec.n_patches,
                       "queries": n_total, "queries_per_gpu": per,
                       "net_boundary_segments": sc.n_net_segments,
                       "parallelism": f"dp{world} (queries sharded, scene replicated, "
                                      "one all-gather)",
                       "l2": "flushed between steps (256 MiB write)"},
            "nominal_pairs_per_s": value * spec.n_patches,
            "candidate_pairs_per_s": stt["candidates"] / (ms_dev * 1e-3 / args.steps) * world,
            "e2e": {"value": e2e, "unit": "queries/s", "h2d_bytes_per_step": int(nq * 24),
                    "d2h_bytes_per_step": int(nq * 9)},
            "e2e_copy_floor": {
                "value": n_total / (ms_cp * 1e-3 / args.steps), "unit": "queries/s",
                "ms_per_step": ms_cp / args.steps, "frac": ms_cp / ms_e2e,
                "note": "the e2e step's input and output copies alone (pinned host memory, "
                        "H2D and D2H concurrently on two streams); frac = floor time / "
                        "e2e time"},
            "gpu_launches": launches,
            "roofline": {"bound": "fp64", "kernel": kname, "achieved": achieved,
                         "peak": peak_tf, "unit": "TFLOP/s",
                         "frac": achieved / peak_tf if peak_tf else None,
                         "traffic": _traffic(kname, args.config, nq),
                         "peak_source": "FP64 DFMA-chain microbenchmark run live on this GPU "
                                        "(MEASURED_PEAKS.json has no FP64 entry)",
                         "kernel_ms": kms, "kernel_share_of_step":
                             kms / (ms_dev / args.steps) if ms_dev else None},
            # the longest kernel of the step is the K2 cull: memory-latency bound,
            # reported against the measured HBM copy bandwidth
            "roofline_cull": _cull_roofline(stt, nq),
            "stage_ms": {"cull": stt["ms_cull"], "k3_candidates": stt["ms_k3_candidates"],
                         "k3_fallback": stt["ms_k3_fallback"], "k3_newton": stt["ms_k3_newton"],
                         "boundary": stt["ms_boundary"], "finalize": stt["ms_other"]},
            "counters": {k: stt[k] for k in ("candidates", "nodes", "newton_iters", "roots",
                                             "k3_newton_items", "k3_fallback_items",
                                             "boundary_segments", "retried", "rounds")},
            "clocks": clock_info,
        }
        if world == 1 and not args.no_ray_reuse:
            out["ray_reuse"] = ray_reuse(G, torch, sc, dev, stream)
        if world == 1 and not args.no_ray_reuse:
            out["roofline_open_scene"] = boundary_roofline(G, torch, dev, stream, peak_tf)
        if world == 1 and not args.no_far_field:
            out["far_field"] = far_field(G, torch, dev, stream)
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(spec, args.cpu_seconds)
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
