"""Benchmark: one FMM evaluate (P2M, M2M, M2L + check->local solve, L2L,
L2P, P2P) of BASELINE config 2 per step - 1M uniform points in [0,1]^3,
charges U[0,1), float32, p=4, depth 5, BLAS-M2L with sigma_min 1e-6.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  ``value`` = evaluate Mpoints/s with the
charges already resident in HBM (device-timed, CUDA events, L2 flushed
between steps); ``e2e`` = the same through the public API
(``FmmInstance.evaluate`` on host charges, H2D + D2H inside the timed
region); ``m2l`` = M2L GFLOP/s from SURVEY 8(d)'s algorithmic flop count;
``roofline`` = the dominant kernel against its measured pipe peak;
``cpu_baseline`` = the reference (Cython-compiled, unmodified) evaluate on
this host's cores.  ``--impl reference`` times that reference alone.
Multi-GPU (torchrun, N>1): the octree is partitioned by level-2 subtrees,
M2L multipole halos are exchanged with NCCL; strong scaling of the same 1M
points (BASELINE metric "1M pts, 1/2/4/8 GPU").
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

if __name__ == "__main__" and any(a.endswith("reference") for a in sys.argv[1:]):
    # Reference arm thread policy: all cores for the OpenMP loops with active
    # waiting (the per-leaf P2M/L2P loops fork ~65k short parallel regions)
    # and single-threaded OpenBLAS (threaded OpenBLAS oversubscribes the
    # cores against the OpenMP team).  Measured on the B200 host (16 cores,
    # c2): this policy 1.70 s/evaluate; PASSIVE 3.73 s; ACTIVE + threaded
    # OpenBLAS 9.98 s; see profiles/r1/README.md.  Must run before numpy loads
    # OpenBLAS (it reads the thread count once, at load).
    _n = str(os.cpu_count() or 1)
    for _k, _v in (("OMP_WAIT_POLICY", "ACTIVE"), ("OMP_NUM_THREADS", _n),
                   ("KIFMM_THREADS", _n), ("OPENBLAS_NUM_THREADS", "1")):
        os.environ.setdefault(_k, _v)

import numpy as np  # noqa: E402  (after the reference-arm thread policy)

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PROFILE_PASSES = 5
METRIC = "M2L GFLOP/s (% roofline) & FMM eval Mpoints/s, Laplace 3D, 1M pts, 1/2/4/8 GPU"
CONFIG = dict(depth=5, order_equiv=4, backend="blas", precision="f32", sigma_min=1e-6)
N_POINTS = 1_000_000
POINT_SEED, CHARGE_SEED = 7, 11


def inputs(n=N_POINTS):
    pts = np.random.default_rng(POINT_SEED).random((n, 3))     # generate_points("uniform-cube")
    q = np.random.default_rng(CHARGE_SEED).random(n)
    return pts, q


def workload(n=N_POINTS):
    return dict(workload="BASELINE config 2: Laplace 3D kiFMM evaluate, N=1,000,000 uniform "
                         "[0,1]^3 sources=targets, charges U[0,1), float32, p=4 (56-point "
                         "surfaces), uniform octree depth 5, BLAS-M2L sigma_min 1e-6, potential",
                n_points=n, seeds={"points": POINT_SEED, "charges": CHARGE_SEED}, **CONFIG)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for s in self.samples for n, v in zip(names, s[2:]) if "Active" in v
                          and "Not" not in v})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ------------------------------------------------------------- work counts
def m2l_flops(inst):
    """per level 2 N_s n_e k + 4 k sum_t m_t k_t + 2 N_t k n_c
    (+ 2 N_t r_d (n_c + n_e) for the solve the reference times inside M2L)."""
    ops = inst.blas_ops
    k = ops.k
    ranks = ops.ranks
    exp = inst.expansions
    n_e, n_c, r_d = exp.n_equiv, exp.n_check, exp.down_inv.rank
    apply_f = solve_f = bucket_f = 0.0
    per_level = {}
    for lvl, b in inst.buckets.items():
        n_s = inst.source_tree.level_keys(lvl).shape[0]
        n_t = inst.target_tree.level_keys(lvl).shape[0]
        bk = sum(4.0 * k * p[0].shape[0] * ranks[i] for i, p in enumerate(b.pairs) if p is not None)
        f = 2.0 * n_s * n_e * k + bk + 2.0 * n_t * k * n_c
        apply_f += f
        bucket_f += bk
        solve_f += 2.0 * n_t * r_d * (n_c + n_e)
        per_level[lvl] = dict(apply=f, bucket=bk, pairs=int(sum(p[0].shape[0] for p in b.pairs
                                                              if p is not None)))
    return apply_f, apply_f + solve_f, per_level


def near_field_counts(inst):
    """P2P work: interactions the reference evaluates (each ordered target /
    near-source pair) and, for sources == targets, the rsqrt the mutual pass
    executes (own-leaf blocks + each adjacent leaf pair once)."""
    near, t = inst.near, inst.target_tree
    n = t.leaf_counts.astype(np.int64)
    owner = np.repeat(np.arange(n.shape[0]), np.diff(near.offsets))
    up = near.leaves > owner
    self_pairs = int((n * n).sum())
    upper_pairs = int((n[owner[up]] * inst.source_tree.leaf_counts[near.leaves[up]]).sum())
    return dict(interactions=int(inst.n_near_pairs), self_pairs=self_pairs,
                upper_pairs=upper_pairs, rsqrt_executed=self_pairs + upper_pairs)


def measured_peaks():
    """Driver-written MEASURED_PEAKS.json, else the profiling guide's fallback."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return dict(hbm_gbs=float(d["hbm_gbs"]), bf16_tflops=float(d["bf16_tflops"]),
                    source="MEASURED_PEAKS.json")
    except Exception:
        return dict(hbm_gbs=6650.0, bf16_tflops=1590.0, source="fallback (B200_PROFILING.md)")


def probe_peak(kind):
    """Measured pipe peak in TFLOP/s (kind 0 FFMA f32, 1 DFMA f64) or
    Gop/s (kind 2, MUFU rsqrt)."""
    import torch
    from paper_2408_07436_b200 import _native as nat
    nat.load()
    blocks, threads, iters = 148 * 8, 256, 4096
    out = torch.empty(blocks * threads, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        nat.call("kifmm_probe", kind, blocks, threads, iters, out.data_ptr(), s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    nat.call("kifmm_probe", kind, blocks, threads, iters, out.data_ptr(), s)
    e1.record()
    torch.cuda.synchronize()
    ops = blocks * threads * iters * 128.0
    sec = e0.elapsed_time(e1) / 1e3
    return (2 * ops / sec / 1e12) if kind != 2 else ops / sec / 1e9


# ------------------------------------------------------------- CPU baseline
def cpu_reference_run(pts, q, steps=1, warmup=0, kw=None):
    """Unmodified reference evaluate (oracle/_ref, Cython-compiled from
    /root/reference) on this host; falls back to the oracle port."""
    kw = kw or CONFIG
    from oracle import reference_available
    cores = os.cpu_count() or 1
    if reference_available():
        from oracle.ref_bridge import make_reference_instance
        inst = make_reference_instance(pts, pts, threads=cores, **kw)
        kind = "reference"
        run = inst.evaluate
    else:
        from oracle import port
        from paper_2408_07436_b200 import FmmConfig, setup
        inst = setup(pts, pts, FmmConfig(**kw))
        kind = "port"
        run = lambda qq: port.evaluate(inst, qq, threads=cores)[:, 0]   # noqa: E731
    for _ in range(warmup):
        run(q)
    times, pot = [], None
    for _ in range(steps):
        t0 = time.perf_counter()
        pot = run(q)
        times.append(time.perf_counter() - t0)
    return dict(kind=kind, cores=cores, times=times, potentials=pot,
                timings=getattr(inst, "timings", {}), instance=inst)


def run_reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    pts, q = inputs()
    steps = max(1, args.steps)
    res = cpu_reference_run(pts, q, steps=steps, warmup=min(args.warmup, 1))
    sec = float(np.mean(res["times"]))
    value = N_POINTS / sec / 1e6
    line = dict(metric=METRIC, value=value, unit="Mpoints/s", impl="reference",
                n_gpus=args.gpus, steps=steps, warmup=min(args.warmup, 1),
                ms_per_step=sec * 1e3, higher_is_better=True, scaling="strong",
                vs_baseline=None, dtype="f32", data="synthetic", config=workload(),
                cpu_baseline=dict(value=value, unit="Mpoints/s", cores=res["cores"],
                                  kind=res["kind"],
                                  sample=f"full workload, {steps} evaluate(s) of 1M points, "
                                         f"threads={res['cores']}, OMP_WAIT_POLICY=ACTIVE, "
                                         "OPENBLAS_NUM_THREADS=1"),
                e2e=dict(value=value, unit="Mpoints/s", h2d_bytes_per_step=0,
                         d2h_bytes_per_step=0),
                m2l_seconds=float(res["timings"].get("m2l", 0.0)),
                operator_seconds={k: float(v) for k, v in res["timings"].items()})
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------- config 3
C3_CONFIG = dict(depth=5, order_equiv=8, backend="fft", precision="f64")


def c3_inputs(n=N_POINTS):
    """BASELINE config 3: the config-2 points, charges U[-1, 1) (seed 11)."""
    pts = np.random.default_rng(POINT_SEED).random((n, 3))
    return pts, np.random.default_rng(CHARGE_SEED).uniform(-1, 1, n)


def run_ref_subprocess(name, out_path):
    """The reference evaluate of a named config in a fresh process: all
    cores for its OpenMP loops with OMP_WAIT_POLICY=ACTIVE (libgomp reads it
    once, at load).  See ref_config_main."""
    n = str(os.cpu_count() or 1)
    env = dict(os.environ, OMP_NUM_THREADS=n, KIFMM_THREADS=n, OMP_WAIT_POLICY="ACTIVE")
    env.pop("OPENBLAS_NUM_THREADS", None)
    r = subprocess.run([sys.executable, os.path.abspath(__file__), "--ref-config", name,
                        "--ref-out", out_path], env=env, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"reference {name} run failed: {r.stderr[-2000:]}")
    return json.loads(r.stdout.strip().splitlines()[-1])


def ref_config_main(name, out_path):
    """Two reference evaluates of one instance: the timed one with
    single-threaded OpenBLAS (the fastest policy measured: it does not
    oversubscribe the cores against the OpenMP team), and one with threaded
    OpenBLAS.  The two differ by BLAS rounding alone, which bounds how
    closely ANY implementation can be said to match "the reference" per
    target (signed charges: near-zero potentials amplify it)."""
    from threadpoolctl import threadpool_limits
    from oracle import reference_available
    pts, q = c3_inputs() if name == "c3" else inputs()
    kw = C3_CONFIG if name == "c3" else CONFIG
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    # setup with threaded LAPACK, as ours (SVD-based operators depend on it)
    if reference_available():
        from oracle.ref_bridge import make_reference_instance
        inst, kind = make_reference_instance(pts, pts, threads=cores, **kw), "reference"
        run = inst.evaluate
    else:
        from oracle import port
        from paper_2408_07436_b200 import FmmConfig, setup
        inst, kind = setup(pts, pts, FmmConfig(**kw)), "port"
        run = lambda qq: port.evaluate(inst, qq, threads=cores)[:, 0]   # noqa: E731
    with threadpool_limits(limits=1, user_api="blas"):
        t1 = time.perf_counter()
        pot = np.asarray(run(q))
        sec = time.perf_counter() - t1
    timings = dict(getattr(inst, "timings", {}))
    pot_mt = np.asarray(run(q))
    np.savez(out_path, timed=pot, blas_threaded=pot_mt)
    print(json.dumps(dict(kind=kind, cores=cores, seconds=sec,
                          total_seconds=time.perf_counter() - t0,
                          operator_seconds={k: float(v) for k, v in timings.items()})))
    return 0


def parity_stats(got, want, tol):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    d = np.abs(got - want)
    rel = d / np.abs(want)
    scale = np.abs(want).max()
    return dict(tol=tol, max_rel=float(rel.max()), strict_failures=int((rel > tol).sum()),
                normwise=float(d.max() / scale),
                floored_max=float((d / np.maximum(np.abs(want), 1e-3 * scale)).max()))


def hadamard_work(inst, lvl):
    """SURVEY 8(d) FFT-M2L algorithmic work at one level, n_rhs = 1:
    F_had = 8 n_freq sum(admissible pairs) flop, B_had = 2 w n_freq
    (N_s + 26 * 64 + N_t) bytes (source spectra, the 26 x 64 kernel
    spectra, target spectra)."""
    ops, plan = inst.fft_ops, inst.halo_plans[lvl]
    kh = np.asarray(ops.khat)
    nz = np.any(kh != 0, axis=0).sum(axis=(1, 2))                 # admissible (tau, sigma) per offset
    pairs = int((nz[None, :] * (np.asarray(plan.halo) >= 0)).sum())
    w = np.dtype(inst.config.dtype).itemsize
    n_s = inst.source_tree.level_keys(lvl).shape[0]
    n_t = inst.target_tree.level_keys(lvl).shape[0]
    return dict(pairs=pairs, flops=8.0 * ops.n_freq * pairs,
                bytes=2.0 * w * ops.n_freq * (n_s + 26 * 64 + n_t))


def run_config3(args, flush, peaks, with_reference=True):
    """BASELINE config 3 on the same GPU: 1M uniform points, charges
    U[-1, 1), float64, p = 8, FFT-M2L, depth 5, potential and gradient."""
    import torch
    from paper_2408_07436_b200 import FmmConfig, setup
    from paper_2408_07436_b200.device import profile_launches
    pts, q = c3_inputs()
    t0 = time.perf_counter()
    inst = setup(pts, pts, FmmConfig(**C3_CONFIG))
    setup_s = time.perf_counter() - t0
    dev = inst.device
    q_dev = torch.from_numpy(q).cuda()
    timed = {}
    for grad in (True, False):
        for _ in range(max(3, args.warmup)):
            dev.evaluate_graphed(q_dev, 1, gradient=grad)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        for e0, e1 in ev:
            flush.zero_()
            e0.record()
            dev.evaluate_graphed(q_dev, 1, gradient=grad)
            e1.record()
        torch.cuda.synchronize()
        timed[grad] = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    flush.zero_()
    with profile_launches() as prof:
        dev.evaluate_device(q_dev, 1, timings=True)
    launches = prof.times()
    per_kernel = {}
    for name, tag, t in launches:
        per_kernel[name.replace("kifmm_", "")] = per_kernel.get(name.replace("kifmm_", ""), 0.0) + t
    lvl = inst.config.depth
    had_ms = sum(t for n, tag, t in launches if "hadamard" in n and tag == f"m2l{lvl}")
    work = hadamard_work(inst, lvl)
    dmma = probe_peak(3)
    had = dict(kernel=f"hadamard_tiled_c128 (level {lvl})", ms=had_ms,
               algorithmic=f"F_had = 8 n_freq sum(pairs) = {work['flops']:.4g} flop, "
                           f"B_had = 2 w n_freq (N_s + 26*64 + N_t) = {work['bytes']:.4g} B "
                           f"(SURVEY 8d), {work['pairs']} admissible pairs",
               fp64_tflops=work["flops"] / (had_ms / 1e3) / 1e12, dmma_peak_tflops=dmma,
               dmma_frac=work["flops"] / (had_ms / 1e3) / 1e12 / dmma,
               hbm_gbs=work["bytes"] / (had_ms / 1e3) / 1e9, hbm_peak_gbs=peaks["hbm_gbs"],
               hbm_frac=work["bytes"] / (had_ms / 1e3) / 1e9 / peaks["hbm_gbs"],
               traffic=dram_traffic("hadamard_tiled_c128_level5"),
               bound="FP64 tensor (DMMA): intensity F_had / B_had ~ 40 flop/B is above the "
                     "DMMA ridge (~5.8 flop/B), so the HBM fraction is reported, not targeted",
               peak_source="kifmm_probe DMMA m8n8k4 measured in this run; HBM "
                           + peaks["source"])
    pot = dev.evaluate_device(q_dev, 1).cpu().numpy()[:, 0].astype(np.float64)
    rec = dict(workload="BASELINE config 3: N=1,000,000 uniform [0,1]^3, charges U[-1,1), "
                        "float64, p=8 (296-point surfaces), FFT-M2L on the 2p grid, depth 5, "
                        "potential and gradient", config=C3_CONFIG, setup_seconds=setup_s,
               ms_per_evaluate_gradient=timed[True], ms_per_evaluate_potential=timed[False],
               value=N_POINTS / (timed[True] / 1e3) / 1e6, unit="Mpoints/s",
               value_potential_only=N_POINTS / (timed[False] / 1e3) / 1e6,
               kernel_ms=per_kernel, hadamard=had,
               timing="CUDA graph replay, CUDA events, L2 flushed between steps")
    if with_reference:
        import tempfile
        with tempfile.TemporaryDirectory() as td:
            path = os.path.join(td, "ref_c3.npz")
            info = run_ref_subprocess("c3", path)
            refs = dict(np.load(path))
        rec["cpu_baseline"] = dict(
            value=N_POINTS / info["seconds"] / 1e6, unit="Mpoints/s", seconds=info["seconds"],
            cores=info["cores"], kind=info["kind"], operator_seconds=info["operator_seconds"],
            sample="one full config-3 evaluate (potential; the reference has no gradient), "
                   "all host threads, OMP_WAIT_POLICY=ACTIVE, single-threaded OpenBLAS")
        rec["parity"] = dict(
            vs_reference=parity_stats(pot, refs["timed"], 1e-10),
            vs_reference_blas_threaded=parity_stats(pot, refs["blas_threaded"], 1e-10),
            reference_vs_itself=parity_stats(refs["timed"], refs["blas_threaded"], 1e-10),
            note="signed charges: near-zero potentials make the per-target ratio depend on "
                 "rounding order alone; the reference's two BLAS threadings disagree by "
                 "reference_vs_itself (SURVEY 8d); full-size records in "
                 "profiles/r2/parity_full")
    return rec


# ------------------------------------------------------------------ ours
def dram_traffic(key):
    """DRAM bytes per launch of a kernel from the committed ncu capture
    (profiles/r2/dram_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2", "dram_traffic.json")) as f:
            return float(json.load(f)[key]["bytes"])
    except (OSError, KeyError, ValueError):
        return None


def run_single(args):
    import torch
    from paper_2408_07436_b200 import FmmConfig, setup
    from paper_2408_07436_b200.device import profile_launches

    torch.cuda.set_device(0)
    pts, q = inputs()
    t0 = time.perf_counter()
    inst = setup(pts, pts, FmmConfig(**CONFIG))
    setup_s = time.perf_counter() - t0
    dev = inst.device
    q_dev = torch.from_numpy(q.reshape(-1, 1)).cuda().reshape(-1)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(args.warmup):
        dev.evaluate_graphed(q_dev, 1)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        for e0, e1 in ev:
            flush.zero_()                      # evict L2 between steps (not timed)
            e0.record()
            dev.evaluate_graphed(q_dev, 1)
            e1.record()
        torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    ms = float(np.mean(step_ms))
    value = N_POINTS / (ms / 1e3) / 1e6

    # per-launch profile (separate, untimed eager passes, L2 flushed before
    # each): the median over PROFILE_PASSES passes of every launch
    passes = []
    for _ in range(PROFILE_PASSES):
        flush.zero_()
        with profile_launches() as prof:
            dev.evaluate_device(q_dev, 1, timings=True)
        passes.append(prof.times())
    launches = [(n, t, float(np.median([p[i][2] for p in passes])))
                for i, (n, t, _) in enumerate(passes[0])]
    phases = dev.collect_timings()
    per_kernel = {}
    for name, tag, t in launches:
        key = name.replace("kifmm_", "")
        per_kernel[key] = per_kernel.get(key, 0.0) + t
    n_launch = len(launches)
    pot_dev = dev.evaluate_device(q_dev, 1).cpu().numpy()[:, 0].copy()

    # M2L GFLOP/s: algorithmic flops over the M2L phases (incl. the solve, as
    # the reference times it)
    f_apply, f_total, per_level = m2l_flops(inst)
    m2l_s = phases.get("m2l", 0.0)
    sweep_t = {t: ms_ for n, t, ms_ in launches if "m2l_sweep" in n}
    # rooflines of the two dominant kernels; `roofline` is the top one
    dom = max(per_kernel.items(), key=lambda kv: kv[1])
    peak_f32 = probe_peak(0)
    peak_mufu = probe_peak(2)                       # Grsqrt/s
    peaks = measured_peaks()
    rooflines = {}
    lvl = inst.config.depth
    bd = dev.blas
    sweep_ms = sweep_t[f"m2l{lvl}"]
    algo = per_level[lvl]["bucket"]
    if bd.tc:
        # 3xTF32 on the TF32 tensor pipe: dense TF32 = bf16 / 2 (same datapath),
        # three MMAs per fp32 product
        peak_tc = peaks["bf16_tflops"] / 2.0 / 3.0
        n_tiles = (dev.tma_plan if dev.tma else dev.blas_plan_dev)[lvl]["n_tiles"]
        clk_mhz = clk.summary().get("sm_mhz") or 1965.0
        smem_peak = 128.0 * 148 * clk_mhz * 1e6 / 1e9                    # GB/s
        tmem = dev.tma and bd.tmem
        kp = bd.kin
        if tmem:
            # tensor-memory sweep (csrc/m2l_tmem.cu): per (tile, vector) one MMA
            # of N = 2 kp (A_hi . [B_hi | B_lo]) and one of N = kp rounded to 16
            # (A_lo . B_hi), K = kp, M = 128; A from TMEM
            n2 = -(-kp // 16) * 16
            execd = 2.0 * 128 * (2 * kp + n2) * kp * 189 * n_tiles
            # shared-memory traffic per (tile, vector): TMA write of the raw
            # source block (128-byte rows, 32-column boxes), the loaders' read
            # of it, half a core pair write (2 tiles per CTA share it), the
            # MMAs' reads of the core pair
            a_b = 128.0 * 128 * (-(-kp // 32))
            smem_bytes = (a_b + 128.0 * kp * 4 + 2.0 * kp * kp * 4 / 2
                          + (2 * kp + n2) * kp * 4.0) * 189 * n_tiles
            kname = "m2l_sweep_tmem_f32"
            note = ("128 B/clk/SM shared-memory bandwidth; TMA source-block write + loader read, "
                    "half a core-pair write, MMA core reads per (tile, vector); A reaches the "
                    "tensor core from TMEM")
        else:
            execd = 3 * 2.0 * 128 * bd.kin * bd.ko_pad * 189 * n_tiles
            # per (tile, vector) TMA writes of A hi/lo + core hi/lo, and the
            # three MMAs' operand reads (A_lo.B_hi, A_hi.B_lo, A_hi.B_hi)
            a_b, b_b = 2 * 4.0 * 128 * bd.kin, 2 * 4.0 * bd.ko_pad * bd.kin
            smem_bytes = (a_b + b_b + 3 * (a_b + b_b) / 2) * 189 * n_tiles
            kname = f"m2l_sweep_{'tma' if dev.tma else 'tc'}_f32"
            note = "128 B/clk/SM shared-memory bandwidth; TMA writes + MMA operand reads per (tile, vector)"
        gather_bytes = 4.0 * bd.kin * per_level[lvl]["pairs"]
        rooflines["m2l_sweep_tc_f32"] = dict(
            bound="tensor",
            kernel=f"{kname} (level {lvl})",
            achieved=algo / (sweep_ms / 1e3) / 1e12, peak=peak_tc, unit="TFLOP/s",
            frac=algo / (sweep_ms / 1e3) / 1e12 / peak_tc,
            traffic=dram_traffic(f"{kname}_level5"),
            smem_model=dict(bytes_per_launch=smem_bytes,
                            achieved_gbs=smem_bytes / (sweep_ms / 1e3) / 1e9,
                            peak_gbs=smem_peak,
                            frac=smem_bytes / (sweep_ms / 1e3) / 1e9 / smem_peak,
                            note=note),
            algorithmic=f"4 k sum_t m_t k_t = {algo:.4g} flop at level {lvl} (SURVEY 8d)",
            executed_tensor_tflops=execd / (sweep_ms / 1e3) / 1e12,
            source_row_gbs=gather_bytes / (sweep_ms / 1e3) / 1e9,
            peak_source="MEASURED_PEAKS.json bf16_tflops / 2 (TF32) / 3 (3xTF32)")
    else:
        rooflines["m2l_sweep"] = dict(
            bound="fp32", kernel=f"m2l_sweep (level {lvl})",
            achieved=algo / (sweep_ms / 1e3) / 1e12, peak=peak_f32, unit="TFLOP/s",
            frac=algo / (sweep_ms / 1e3) / 1e12 / peak_f32, traffic=None,
            algorithmic=f"4 k sum_t m_t k_t = {algo:.4g} flop at level {lvl}",
            peak_source="kifmm_probe FFMA measured in this run")
    inter = inst.n_near_pairs
    l2p = float(inst.target_tree.n_points) * inst.expansions.n_equiv
    nf = near_field_counts(inst)
    if "p2p_mutual_f32" in per_kernel:
        # mutual near field: every adjacent leaf pair once (one rsqrt, both
        # directions) + the own-leaf blocks; L2P runs in l2p_mutual_f32
        leaf_key = "p2p_mutual_f32"
        leaf_ms = per_kernel[leaf_key]
        execd = nf["rsqrt_executed"]
        rooflines[leaf_key] = dict(
            bound="mufu", kernel=leaf_key, achieved=execd / (leaf_ms / 1e3) / 1e9,
            peak=peak_mufu, unit="Grsqrt/s", frac=execd / (leaf_ms / 1e3) / 1e9 / peak_mufu,
            traffic=dram_traffic("p2p_mutual_f32"),
            algorithmic=f"{inter} P2P interactions served by {execd} executed rsqrt "
                        f"({nf['self_pairs']} own-leaf + {nf['upper_pairs']} mutual pairs)",
            interactions_per_s=inter / (leaf_ms / 1e3),
            rsqrt_executed=execd, interactions=inter,
            tflops_11_per_interaction=11.0 * inter / (leaf_ms / 1e3) / 1e12, fp32_peak=peak_f32,
            peak_source="kifmm_probe MUFU.RSQ measured in this run")
    else:
        leaf_key = [k for k in per_kernel if k.startswith("leaf_pass")][0]
        leaf_ms = per_kernel[leaf_key]
        rooflines[leaf_key] = dict(
            bound="mufu", kernel=leaf_key, achieved=(inter + l2p) / (leaf_ms / 1e3) / 1e9,
            peak=peak_mufu, unit="Grsqrt/s", frac=(inter + l2p) / (leaf_ms / 1e3) / 1e9 / peak_mufu,
            traffic=dram_traffic("leaf_pass_f32"),
            algorithmic=f"{inter} P2P + {l2p:.0f} L2P kernel evaluations (one rsqrt each)",
            rsqrt_executed=inter + l2p, interactions=inter,
            tflops_11_per_interaction=11.0 * inter / (leaf_ms / 1e3) / 1e12, fp32_peak=peak_f32,
            peak_source="kifmm_probe MUFU.RSQ measured in this run")
    roof = rooflines["m2l_sweep_tc_f32" if bd.tc else "m2l_sweep"] if "sweep" in dom[0] \
        else rooflines[leaf_key]

    # e2e through the public API (host charges in pinned memory -> host potentials)
    q_pinned = torch.from_numpy(q).pin_memory().numpy()
    # warm-up until the caching host allocator holds the pinned result buffers
    # (a caller keeps the previous result alive while the next one is made)
    # and with an ordinary (pageable) numpy array, as reference callers pass
    q_page = np.array(q, copy=True)
    # warm-up of both paths: until the caching host allocator holds the pinned
    # result buffers (a caller keeps the previous result alive while the next
    # one is made) and the host cores run at speed
    out = None
    for _ in range(max(20, args.warmup)):
        out = inst.evaluate(q_pinned)
        inst.evaluate(q_page)

    def e2e_batch(qh, n):
        ts, res = [], None
        for _ in range(n):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = inst.evaluate(qh)
            ts.append(time.perf_counter() - t0)
        return float(np.mean(ts)), res

    # mean seconds per call of the best of 3 batches of >= 20 calls per input
    # kind, the kinds alternating (a host hiccup - page faults, a pinned
    # allocation - in one call otherwise sets the number, and whichever kind
    # is measured first on a cold host loses)
    n_calls = max(20, args.steps)
    best = {"pinned": None, "pageable": None}
    for _ in range(3):
        for kind, qh in (("pinned", q_pinned), ("pageable", q_page)):
            m, res = e2e_batch(qh, n_calls)
            best[kind] = m if best[kind] is None else min(best[kind], m)
            if kind == "pinned":
                out = res
    e2e_s = best["pinned"]
    e2e_t = [e2e_s] * n_calls
    e2e_value = N_POINTS / e2e_s / 1e6
    e2e_pageable = N_POINTS / best["pageable"] / 1e6

    # CPU baseline (reference, bounded sample: one full evaluate) + parity of this run
    cpu = None
    if not args.no_cpu_baseline:
        res = cpu_reference_run(pts, q, steps=1)
        csec = min(res["times"])
        ref = np.asarray(res["potentials"], dtype=np.float64)
        rel = np.abs(out.astype(np.float64) - ref) / np.abs(ref)
        cpu = dict(value=N_POINTS / csec / 1e6, unit="Mpoints/s", cores=res["cores"],
                   kind=res["kind"], sample="one full 1M-point evaluate, all host threads "
                   "(in the bench process; default thread policy)", seconds=csec,
                   operator_seconds={k: float(v) for k, v in res["timings"].items()},
                   parity_max_rel=float(rel.max()), parity_tol=1e-5)
    c3 = None
    if not args.no_config3:
        c3 = run_config3(args, flush, peaks, with_reference=not args.no_cpu_baseline)
    line = dict(metric=METRIC, value=value, unit="Mpoints/s", n_gpus=1, steps=args.steps,
                warmup=args.warmup, ms_per_step=ms, higher_is_better=True, scaling="strong",
                vs_baseline=None, dtype="f32", data="synthetic (seeded; no dataset involved)",
                config=dict(workload(), l2="flushed between steps (256 MB write)",
                            execution="whole evaluate captured as one CUDA graph; "
                                      "per-kernel times: median of 5 eager passes (CUDA events)",
                            parallelism="1 GPU"),
                m2l=dict(gflops=f_total / m2l_s / 1e9 if m2l_s else None,
                         seconds=m2l_s, flops_apply=f_apply, flops_with_solve=f_total),
                operator_seconds=phases, kernel_ms=per_kernel, roofline=roof,
                roofline_all=rooflines,
                cpu_baseline=cpu,
                e2e=dict(value=e2e_value, unit="Mpoints/s", calls=len(e2e_t),
                         timing="mean seconds per call of the best of 3 batches of calls "
                                "(pinned and pageable batches alternating, after 20 warm-up "
                                "calls of each), host wall clock, synchronised before every call",
                         host_input="pinned float64 charges (pageable_value: an ordinary "
                                    "numpy array, as reference callers pass)",
                         pageable_value=e2e_pageable,
                         h2d_bytes_per_step=int(q.nbytes),
                         d2h_bytes_per_step=int(out.nbytes)),
                gpu_launches=n_launch * args.steps, clocks=clk.summary(),
                setup_seconds=setup_s, p2p_interactions=inst.n_near_pairs,
                configs={"c3": c3} if c3 is not None else {})
    print(json.dumps(line), flush=True)
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-config3", action="store_true",
                    help="skip the config-3 (FFT-M2L, float64) extra measurement")
    ap.add_argument("--ref-config", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--ref-out", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--force-dist", action="store_true",
                    help="use the partitioned (torchrun) path even for one rank")
    args = ap.parse_args(argv)
    if args.ref_config:
        return ref_config_main(args.ref_config, args.ref_out)
    if args.impl == "reference":
        return run_reference_arm(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1 or args.force_dist:
        from paper_2408_07436_b200 import distributed
        return distributed.bench_main(args, sys.modules[__name__])
    return run_single(args)


if __name__ == "__main__":
    sys.exit(main())
