#!/usr/bin/env python
"""Benchmark of the Paralpha hot path: one alpha-circulant preconditioned Richardson iteration
(arXiv 2103.12571) per step, metric = space-time unknowns updated per second (L*M*N / t_iter).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl pint|reference]

N > 1 is launched by torchrun (one process per GPU).  Default workload: BASELINE.json config 5
(2-D advection 1024^2, M=4, L=512; 2.1e9 unknowns, 34.4 GB per vector — fits one B200).
Prints ONE JSON line on rank 0.  See DESIGN.md §6 for the measurement recipe.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "space-time unknowns updated/s per Richardson iteration (fp64), 1/2/4/8 B200, % HBM roof"
UNIT = "unknowns/s"

# algorithmic HBM bytes per unknown of each launch (compulsory reads + writes)
ALGO_BYTES = {"fwd_kernel": 32, "pcr_classes_kernel": 32, "pcr_chunk_kernel": 32, "fft2d_rows_kernel<fwd>": 32,
              "fft2d_cols_kernel": 32, "fft2d_rows_kernel<inv>": 32, "bwd_kernel": 48, "residual2d_kernel": 32,
              "tfft_fwd_kernel": 32, "tfft_bwd_kernel": 48,
              # persistent 2-D spatial pipeline: the three plane passes' compulsory traffic (3 x 32 B)
              "spatial2d_kernel": 96,
              # pipelined plane passes (same 3 x 32 B, one launch each)
              "rows_pipe_kernel<fwd>": 32, "cols_pipe_kernel": 32, "rows_pipe_kernel<inv>": 32,
              # pipelined time transforms (forward in place, inverse x2 + u -> u)
              "tfft_pipe_kernel<fwd>": 32, "tfft_pipe_kernel<inv>": 48,
              # TMA-staged time tiles (the inverse's u += c is a TMA reduce-add at the L2: u is still read
              # and written once in HBM)
              "tfft_fwd_tma_kernel": 32, "tfft_bwd_tma_kernel": 48,
              # fused R / C / I plane passes (one launch; compulsory 3 x 32 B, L2 reuse can only lower it)
              "spatial_fused_kernel": 96,
              # 1-D pipelined passes (TMA forward tile, two-pass PCR)
              "fwd1d_tma_kernel": 32, "pcr_cls_pipe_kernel": 32, "pcr_chunk_pipe_kernel": 32,
              # generic-grid path (paper's Table 1/2 sizes): one read + one write per pass
              "resid_any_kernel": 32, "node_any_kernel<Sinv>": 32, "fft_any_kernel<fwd x>": 32,
              "fft_any_kernel<fwd y>": 32, "divide_any_kernel": 32, "fft_any_kernel<inv y>": 32,
              "fft_any_kernel<inv x>": 32, "node_any_kernel<SG>": 32}
# direct form (u = C_a^{-1}((C_a - C)u + w)): no read of u, input synthesized from one N-vector
ALGO_BYTES_DIRECT = {"direct_r0_kernel": 0, "plane_rows_dif_kernel": 0, "plane_cols_dif_kernel": 0,
                     "spec_blocked_kernel": 0, "cols_direct_kernel": 16, "cols_pipe_kernel<synth>": 16,
                     "fft2d_rows_kernel<inv>": 32, "rows_pipe_kernel<inv>": 32, "tfft_bwd_kernel": 32,
                     "pcr_classes_kernel": 16, "pcr_chunk_kernel": 32, "bwd_kernel": 32,
                     "spatial2d_kernel": 48, "tfft_pipe_kernel<inv>": 32,
                     "tfft_bwd_tma_kernel": 32}
# real-data (Hermitian) mode: u stored as real fp64 (8 B per unknown), time series packed two real
# points per complex value (8 B per unknown), L/2 + 1 of the L frequencies solved (unit planes:
# 8 B per unknown, up to a factor 1 + 2/L)
ALGO_BYTES_HERM = {"residual2d_kernel": 16, "tfft_fwd_kernel": 16, "rows_pipe_kernel<fwd>": 16,
                   "cols_pipe_kernel": 16, "rows_pipe_kernel<inv>": 16, "tfft_bwd_kernel": 24,
                   "spatial2d_kernel": 48, "fwd_kernel": 16, "fwd1d_tma_kernel": 16, "pcr_classes_kernel": 16,
                   "pcr_chunk_kernel": 16, "pcr_cls_pipe_kernel": 16, "pcr_chunk_pipe_kernel": 16,
                   "bwd_kernel": 24}
ALGO_BYTES_HERM_DIRECT = {"direct_r0_kernel": 0, "plane_rows_dif_kernel": 0, "plane_cols_dif_kernel": 0,
                          "spec_blocked_kernel": 0, "cols_pipe_kernel<synth>": 8, "rows_pipe_kernel<inv>": 16,
                          "tfft_bwd_kernel": 16, "spatial2d_kernel": 24, "pcr_classes_kernel": 8,
                          "pcr_chunk_kernel": 16, "bwd_kernel": 16}


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def schedule_for(p, w_inf, n):
    """The config's alpha sequence (fixed, or Algorithm 2 from the library), repeated to length n."""
    import paper_2103_12571_b200 as P
    if p.alpha_mode == "fixed":
        base = [p.alpha_fixed] * p.iters
    else:
        base = list(P.adaptive_schedule(p.L, w_inf, p.m0, p.iters, p.eps, p.tau)[0])
    return [base[i % len(base)] for i in range(n)]


def cpu_oracle_rate(p, target_s: float, seed: int = 0):
    """The oracle (oracle/paralpha.py ModeOracle, as it stands) on a bounded sample of the workload:
    a random subset of the spatial Fourier modes (each an independent L*M-unknown subproblem of the
    same iteration), one iteration with the config's first alpha.  Returns (unknowns/s, sample text, s)."""
    from oracle.paralpha import ModeOracle, mode_coefficients
    from oracle.schedule import adaptive_schedule
    u0 = p.u0()
    if p.alpha_mode == "fixed":
        a = p.alpha_fixed
    else:
        a = adaptive_schedule(p.L, float(np.abs(u0).max()), p.m0, 1, p.eps, p.tau)[0][0]
    rng = np.random.default_rng(seed)

    def run(nmodes):
        kx = rng.integers(0, p.nx, nmodes)
        ky = rng.integers(0, p.ny, nmodes)
        t0 = time.perf_counter()
        uh0 = mode_coefficients(p, u0, kx, ky)       # the spatial projection of u0 (timed too)
        mo = ModeOracle(p, uh0, kx, ky)
        uh = mo.initial()
        mo.iterate(uh, a)
        return time.perf_counter() - t0

    n = 16
    dt = run(n)
    while dt < target_s / 4 and n < p.N:
        n = min(p.N, n * 4)
        dt = run(n)
    rate = p.L * p.M * n / dt
    return rate, (f"{n} of {p.N} spatial Fourier modes x all L*M={p.L * p.M} (one iteration, ModeOracle, "
                  f"projection of u0 onto the sampled modes included)"), dt


def host_info():
    """CPU model and the BLAS numpy uses (for the cpu_baseline record)."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        libs = [f"{i.get('internal_api')} {i.get('version')} ({i.get('num_threads')} threads)"
                for i in threadpool_info() if i.get("user_api") == "blas"]
        blas = "; ".join(libs) or None
    except Exception:
        pass
    return {"cpu_model": model, "blas": blas, "host_cores": len(os.sched_getaffinity(0))}


def threads_used():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return len(os.sched_getaffinity(0))


def run_reference(args, p, rank, world):
    """--impl reference: the CPU oracle as it stands, on this arm's config/metric (rank 0 only)."""
    if rank != 0:
        return None
    per_step = []
    sample = ""
    for i in range(args.warmup + args.steps):
        rate, sample, dt = cpu_oracle_rate(p, target_s=args.ref_step_s, seed=i)
        if i >= args.warmup:
            per_step.append((rate, dt))
    rates = [r for r, _ in per_step]
    value = float(np.median(rates))
    cores = threads_used()
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": float(np.median([d for _, d in per_step]) * 1e3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128 (fp64)",
            "data": "synthetic (workloads.py seeded generators)", "impl": "reference",
            "config": {"workload": p.name, "cfg": args.config, "L": p.L, "M": p.M, "N": p.N,
                       "unknowns": p.U},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             **host_info()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="pint", choices=["pint", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-target-s", type=float, default=15.0)
    ap.add_argument("--ref-step-s", type=float, default=6.0)
    ap.add_argument("--grid", type=int, default=0, help="profiling only: override nx (and ny in 2-D)")
    ap.add_argument("--form", default="correction", choices=["correction", "direct"],
                    help="iteration form: correction (north star, default) or direct (Alg. 1 as printed)")
    ap.add_argument("--no-sequential", action="store_true", help="skip the sequential Radau IIA baseline")
    ap.add_argument("--hermitian", action="store_true",
                    help="real-data fast path (SURVEY 8(f) row 1): solve only frequencies k <= L/2")
    ap.add_argument("--graph", action="store_true", help="also time CUDA-graph replays (fixed-alpha configs)")
    ap.add_argument("--allow-experiments", action="store_true",
                    help="A/B only: accept a library built with -DPINT_EXPERIMENTS (PINT_LIBRARY)")
    args = ap.parse_args()
    rank, world, local = env_rank()
    p = W.CONFIGS[args.config]
    if args.grid:
        p = p.replace(name=p.name + f"_grid{args.grid}", nx=args.grid, ny=args.grid if p.dim == 2 else 1)

    if args.impl == "reference":
        line = run_reference(args, p, rank, world)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    import torch
    import paper_2103_12571_b200 as P
    experiments = P.experiments_enabled()
    if experiments and not args.allow_experiments:
        sys.exit("bench.py: the loaded libpint was built with -DPINT_EXPERIMENTS (environment switches); "
                 "refusing to report it (pass --allow-experiments for A/B runs)")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    u0 = p.u0()
    if world > 1:
        # time-sharded across the ranks (cyclic steps, four-step FFT, NCCL all-to-all + ring halo)
        from paper_2103_12571_b200.distributed import sharded_solver
        s = sharded_solver(p, u0, device=local)
    else:
        # a dedicated (non-default) stream: the CUDA-graph leg captures the library's launches on it
        s = P.Solver(p, u0, device=local, stream=torch.cuda.Stream(device=local))
    if args.form != "correction":
        s.set_form(args.form)
    if args.hermitian:
        if world > 1:
            sys.exit("bench.py: --hermitian is single-rank (the real-data mode is not built for time-sharded ranks)")
        s.set_hermitian(True)
    stream = s.stream
    w_inf = s.w_inf()
    nlaunch = s.launches_per_iteration()
    names = s.kernel_names()

    # ---- device-timed region: W warm-up + K timed iterations, inputs resident in HBM ----------
    s.set_alpha_schedule(schedule_for(p, w_inf, min(64, args.warmup + args.steps)))
    for _ in range(args.warmup):
        s.iterate(1)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def roll(seconds):
        """Untimed iterations of the same workload for `seconds` (clock window of short regions)."""
        t_end = time.perf_counter() + seconds
        while time.perf_counter() < t_end:
            s.set_alpha_schedule(schedule_for(p, w_inf, 8))
            s.iterate(8)
            torch.cuda.synchronize()

    with ClockSampler(local) as clk:
        # a timed region shorter than the sampler's period cannot be sampled alone: then the window
        # is the timed region plus 0.5 s of the same iterations before and after (recorded below)
        short = p.U < 1e9
        if short:
            roll(0.5)
            s.set_alpha_schedule(schedule_for(p, w_inf, min(64, args.steps)))
            barrier()
        ev0.record(stream)
        done = 0
        while done < args.steps:
            n = min(args.steps - done, (64 - args.warmup if not short else 64) if done == 0 else 64)
            if done > 0:
                s.set_alpha_schedule(schedule_for(p, w_inf, n))  # only for K > 61 (host work, re-timed)
            s.iterate(n)
            done += n
        ev1.record(stream)
        torch.cuda.synchronize()
        if short:
            roll(0.5)
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1)) / args.steps
    value = p.U / (ms * 1e-3)          # the whole problem (all ranks together) per iteration

    # ---- per-kernel device times (same kernels, events after every launch; 1 rank only) -------
    peak, peak_src = measured_peaks()
    phases = None
    if world == 1:
        nprof = max(3, min(args.steps, 10))
        s.set_alpha_schedule(schedule_for(p, w_inf, nprof + 1))
        s.iterate(1)
        kms = s.iterate_profiled(nprof)
    else:
        kms = None
        # communication / computation split of the overlapped schedule (events around the phases
        # of one iteration on every rank, max over ranks)
        s.set_phase_timing(True)
        s.set_alpha_schedule(schedule_for(p, w_inf, 2))
        s.iterate(1)
        ph = s.phase_times()
        s.set_phase_timing(False)
        phases = {k: max_over_ranks(v) for k, v in ph.items()}
    algo_tab = dict(ALGO_BYTES_DIRECT if args.form == "direct" else ALGO_BYTES)
    if args.hermitian:
        algo_tab.update(ALGO_BYTES_HERM_DIRECT if args.form == "direct" else ALGO_BYTES_HERM)
    unknown = [n_ for n_ in names if n_ not in algo_tab]
    if unknown:   # every launch of the iteration needs its byte model (no silent default)
        sys.exit(f"bench.py: no algorithmic byte model for {unknown} (form {args.form}, hermitian {args.hermitian})")
    model_bytes = sum(algo_tab[n_] for n_ in names)
    iteration_roof = {"model_bytes_per_unknown": model_bytes,
                      "achieved_gbs": model_bytes * p.U / world / (ms * 1e-3) / 1e9,
                      "frac": model_bytes * p.U / world / (ms * 1e-3) / 1e9 / peak,
                      "floor96_frac": 96 * p.U / world / (ms * 1e-3) / 1e9 / peak,
                      "note": "per GPU (local share of the HBM model bytes)"}
    if kms is None:
        roofline = {"bound": "hbm", "kernel": None, "achieved": iteration_roof["achieved_gbs"], "peak": peak,
                    "unit": "GB/s", "frac": iteration_roof["frac"], "traffic": None, "peak_source": peak_src,
                    "iteration": iteration_roof, "note": "multi-rank: per-launch profiling is single-rank only"}
    top = int(np.argmax(kms)) if kms is not None else 0
    top_name = names[top]
    algo = algo_tab[top_name] * p.U
    achieved = algo / (kms[top] * 1e-3) / 1e9 if kms is not None else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(p.name, {}).get(top_name)
        except Exception:
            traffic = None
    if kms is not None:
        roofline = {"bound": "hbm", "kernel": top_name, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                    "algo_bytes_per_launch": algo,
                    "kernel_share_of_step": float(kms[top] / kms.sum()),
                    "per_kernel_ms": {n_: float(v) for n_, v in zip(names, kms)},
                    "iteration": iteration_roof}

    # ---- launch-bound configs: the same iteration replayed from a CUDA graph (fixed alpha) ---------
    graph = None
    if world == 1 and (args.graph or (p.alpha_mode == "fixed" and ms < 1.0)) and p.alpha_mode == "fixed":
        ng = 16
        s.set_alpha_schedule(schedule_for(p, w_inf, 64))
        s.iterate(1)
        torch.cuda.synchronize()
        gr = s.graph_create(ng)              # ng iterations captured by the library on its stream
        reps = max(3, args.steps)
        s.graph_launch(gr)
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(reps):
            s.graph_launch(gr)
        g1.record(stream)
        torch.cuda.synchronize()
        s.graph_destroy(gr)
        gus = g0.elapsed_time(g1) * 1e3 / (reps * ng)
        graph = {"us_per_iteration": gus, "value": p.U / (gus * 1e-6), "unit": UNIT, "iterations_per_graph": ng,
                 "replays": reps, "what": "16 iterations captured in one CUDA graph by pint_graph_create on the library stream "
                 "(fixed alpha: every replay is 16 more iterations), device-timed replays"}

    # ---- end to end through the public API with host buffers -----------------------------------
    e2e = None
    if not args.no_e2e:
        u0_pin = torch.from_numpy(u0.view(np.float64).copy()).pin_memory()
        out_pin = torch.empty(2 * p.N, dtype=torch.float64).pin_memory()
        u0_np = u0_pin.numpy()
        out_np = out_pin.numpy()
        s.set_alpha_schedule(schedule_for(p, w_inf, min(64, args.warmup + args.steps)))
        ke = min(args.steps, 64 - args.warmup)

        def e2e_step():
            s.set_initial_value(u0_np.view(np.complex128), reset=False)   # H2D of the step's input
            s.iterate(1)
            s.get_final_value(out_np.view(np.complex128))                 # D2H of the result (syncs)

        for _ in range(args.warmup):
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(ke):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        ems = max_over_ranks(max(e0.elapsed_time(e1), wall * 1e3)) / ke
        e2e = {"value": p.U / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 16 * p.N * world,
               "d2h_bytes_per_step": 16 * p.N, "ms_per_step": ems,
               "what": "per step: H2D u0 (pinned) -> pint_iterate(1) -> D2H u_{L-1,M-1} (solution at T)"}

    # ---- sequential Radau IIA baseline on the same GPU (1 rank) -------------------
    seq = None
    pow2 = all(v & (v - 1) == 0 for v in (p.nx, p.ny))
    if world == 1 and pow2 and not args.no_sequential:
        if args.hermitian:
            s.set_hermitian(False)                       # the sequential baseline uses complex storage
        s.sequential()                                   # warm-up
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s.sequential()
        e1.record(stream)
        torch.cuda.synchronize()
        sms_ = e0.elapsed_time(e1)
        if args.hermitian:
            s.set_hermitian(True)
        s.set_initial_value(u0, reset=True)
        tol = 1e-10 * float(np.abs(u0).max())
        r = s.solve(p.m0, tol, 40, p.eps, p.tau)        # Algorithm 2 to tol (host-timed, not the metric)
        seq = {"ms": sms_, "steps": p.L, "per_step_ms": sms_ / p.L,
               "paralpha_iterations_to_tol": r["iters"], "tol_rel": 1e-10, "stop": r["stop"],
               "paralpha_time_to_tol_ms": r["iters"] * ms,
               "what": ("pint_sequential: L collocation steps, each M shifted spatial solves on the same kernels "
                        "(2-D: FFT-diagonal; 1-D: PCR)")}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, sample, _ = cpu_oracle_rate(p, target_s=args.cpu_target_s)
        cpu = {"value": rate, "unit": UNIT, "cores": threads_used(), "kind": "oracle", "sample": sample, **host_info()}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong" if world > 1 else "weak",
                "vs_baseline": None, "dtype": "c128 (fp64)",
                "data": "synthetic (workloads.py seeded generators; BASELINE.json config recipe)",
                "config": {"workload": p.name, "cfg": args.config, "L": p.L, "M": p.M, "N": p.N,
                           "unknowns": p.U, "bytes_per_vector": 16 * p.U, "form": args.form,
                           "hermitian": bool(args.hermitian),
                           "library": "experiments (A/B build)" if experiments else "product",
                           "l2": "inputs larger than L2 (no flush)" if 16 * p.U > 126e6 else "L2-resident",
                           "parallelism": "single GPU" if world == 1 else
                           f"time-sharded over {world} GPUs (cyclic steps, four-step FFT, NCCL all-to-all + ring halo)"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "sequential_baseline": seq,
                "phases_ms": phases,
                "gpu_launches": (nlaunch if world == 1 else nlaunch + 3) * args.steps,
                "clocks": {**clk.summary(), "window": ("timed region +- 0.5 s of the same iterations"
                                                       if p.U < 1e9 else "timed region")},
                "graph": graph}
        print(json.dumps(line), flush=True)
    s.close()
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
