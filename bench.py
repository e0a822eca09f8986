"""Benchmark of the B200-native mini-BA (BASELINE.json metric: mini-BA
problems/sec and LM iterations/sec, % of HBM roofline, vs the CPU reference).

    python bench.py [--gpus N --steps K --warmup W] [--config 1..5] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU)

A step is one full mba_solve launch over this rank's shard of the workload
(every problem solved from its initial parameters to termination). Problems
are independent: the batch is sharded contiguously over ranks with no
collective on the data path; the per-problem summaries are all-gathered at the
end of each step (the "final gather"). Default workload: BASELINE config 4
(65,536 problems of 8 frames x K=2,000), whose inputs (2.1 GB) exceed L2.

`--impl reference` times the CPU reference path (the oracle port of
miniba.py:223-296, oracle/miniba_oracle.py) on all host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
for _p in (REPO, os.path.join(REPO, "src")):
    if _p not in sys.path:
        sys.path.insert(0, _p)

METRIC = "mini-BA problems/sec and LM iters/sec; % of HBM roofline; vs CPU ref"
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12   # derived nominal
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12    # derived nominal (64 DFMA lanes / SM / clk)
KERNEL_NAME = "mba::v4::solve_v4_kernel (cluster-resident; + mba::solve_kernel launch for plan overflows)"


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh).get("hbm_gbs", 6559.7), "measured"
    except OSError:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# workload

def workload(cfg_id, n_override=None):
    from paper_2506_05558_b200.synth import CONFIGS
    c = dict(CONFIGS[cfg_id])
    if n_override:
        c["n_problems"] = n_override
    return c


def make_shard(c, first, count, seed=0, workers=1):
    from paper_2506_05558_b200.synth import make_batch
    return make_batch(count, n_cams=c["n_cams"], K=c["K"], seed=seed,
                      outlier_frac=c.get("outlier_frac", 0.0), first=first, workers=workers)


def algorithmic_work(batch, n_iters, evals, fused=False):
    """Bytes and flops per SURVEY 8d from the executed evals trace, counting
    only the passes the kernel executes, each at its algorithmic minimum:
    bytes = sum_problems [16K + 12P + sum_it passes_it (16K + 24P)]
    flops per iteration ~ 340K + sum_p[40 + 24C_p + 3C_p(C_p+1)] + C^3/3 + 2C^2
                          + trials_it (40K + sum_p (6C_p + 18)),  C_p = 6 * free cams seeing p + 1.
    Sequential kernels: passes = 1 + n_eval. The cluster-resident kernel
    (fused=True) evaluates try 0 alone and tries 1..4 in one fused pass:
    passes = 1 + [n_eval >= 1] + [n_eval >= 2]. Trial flops count the reference's
    n_eval in both cases."""
    B = batch.n_problems
    K = np.diff(batch.obs_off).astype(np.float64)
    P = np.diff(batch.pt_off).astype(np.float64)
    live = np.arange(evals.shape[1])[None, :] < np.asarray(n_iters)[:, None]
    ev = evals.astype(np.float64) * live
    if fused:
        n_pass_sum = ((ev >= 1).astype(np.float64) + (ev >= 2)).sum(axis=1)
    else:
        n_pass_sum = ev.sum(axis=1)
    # flops: only the trial evaluations the reference performs (b + 1 for an
    # accept at 2^-b, 5 for a rejection), not the fused pass's speculative ones
    n_eval_sum = ev.sum(axis=1)
    passes = np.asarray(n_iters, dtype=np.float64) + n_pass_sum
    bytes_ = float(np.sum(16 * K + 12 * P + passes * (16 * K + 24 * P)))
    # per-point camera multiplicity (free cameras only) -> C_p
    free_obs = ~batch.fixed[batch.cam_off[:-1].repeat(np.diff(batch.obs_off)) + batch.cam]
    gpt = np.repeat(batch.pt_off[:-1], np.diff(batch.obs_off)) + batch.pt
    ncam_p = np.bincount(gpt[free_obs], minlength=int(batch.pt_off[-1])).astype(np.float64)
    Cp = 6 * ncam_p + 1
    prob_of_pt = np.repeat(np.arange(B), np.diff(batch.pt_off))
    schur_p = np.bincount(prob_of_pt, weights=40 + 24 * Cp + 3 * Cp * (Cp + 1), minlength=B)
    trial_p = np.bincount(prob_of_pt, weights=6 * Cp + 18, minlength=B)
    nfree = np.array([np.count_nonzero(~batch.fixed[batch.cam_off[b]:batch.cam_off[b + 1]])
                      for b in range(B)], dtype=np.float64)
    C = 6 * nfree + 1
    iters = n_iters.astype(np.float64)
    flops = float(np.sum(iters * (340 * K + schur_p + C ** 3 / 3 + 2 * C ** 2)
                         + n_eval_sum * (40 * K + trial_p)))
    return bytes_, flops


# ---------------------------------------------------------------------------
# clocks during the timed region (pynvml)

class ClockSampler:
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.index, self.samples, self.reasons, self._stop = index, [], set(), False
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop:
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop = True
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# CPU reference timing (oracle port of the reference path)

def _cpu_solve(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    c, idx, seed, max_iters = args
    from oracle import miniba_oracle as O
    b = make_shard(c, idx, 1, seed=seed)
    p = b.problem(0)
    t0 = time.perf_counter()
    info = O.lm(p, max_iters=max_iters, loss=c["loss"])
    return time.perf_counter() - t0, len(info["accepted"])


def cpu_reference(c, budget_s=15.0, seed=0, steps=1, warmup=0):
    """Solve problems 0, 1, 2, ... of the workload on all host cores (one
    worker process per core, OPENBLAS_NUM_THREADS=1): `warmup` untimed steps
    of one problem per core, then `steps` timed steps of about budget_s /
    steps seconds each, continuing through the problem sequence. Returns
    (problems/s, iterations/s, cores, sample, seconds, per-step seconds)."""
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    if c["n_problems"] == 1 and c["K"] >= 100000:
        # one stress problem: a full 50-iteration CPU solve takes ~20 min, so
        # time the first 2 LM iterations on one core and scale to the solve
        _pool_init()
        sec, it = _cpu_solve((c, 0, seed, 2))
        ips = it / sec
        return (ips / c["max_iters"], ips, 1, f"first 2 LM iterations of the single problem, 1 core "
                f"({sec:.1f} s); problems/s = iterations/s / {c['max_iters']}", sec, [sec])
    ctx = mp.get_context("spawn")
    nxt = 0
    with ctx.Pool(cores, initializer=_pool_init) as pool:
        def run(budget, min_jobs):
            nonlocal nxt
            done = iters = 0
            t0 = time.perf_counter()
            pending = []
            while True:
                while (len(pending) < 2 * cores and nxt < c["n_problems"]
                       and (done + len(pending) < min_jobs or time.perf_counter() - t0 < budget)):
                    pending.append(pool.apply_async(_cpu_solve, ((c, nxt, seed, c["max_iters"]),)))
                    nxt += 1
                if not pending:
                    break
                r = pending.pop(0).get()
                done += 1
                iters += r[1]
            return done, iters, time.perf_counter() - t0
        for _ in range(warmup):
            run(0.0, cores)
        first = nxt
        per_step = max(1.0, budget_s / max(steps, 1))
        # timed steps: the pool stays full across step boundaries (no drain
        # between steps); a step is a per_step-second window and counts the
        # solves completed in it
        tot = []
        pending = []
        t_prev = time.perf_counter()
        for s_ in range(max(steps, 1)):
            t_end = t_prev + per_step
            done = iters = 0
            last = s_ == max(steps, 1) - 1
            while True:
                while len(pending) < 2 * cores and nxt < c["n_problems"] and time.perf_counter() < t_end:
                    pending.append(pool.apply_async(_cpu_solve, ((c, nxt, seed, c["max_iters"]),)))
                    nxt += 1
                if not pending or (not last and time.perf_counter() >= t_end and not pending[0].ready()):
                    break
                r = pending.pop(0).get()
                done += 1
                iters += r[1]
            now = time.perf_counter()
            tot.append((done, iters, now - t_prev))
            t_prev = now
    done = sum(t[0] for t in tot)
    iters = sum(t[1] for t in tot)
    el = sum(t[2] for t in tot)
    used = min(cores, max(done, 1))
    sample = (f"problems {first}..{first + done - 1} of the workload in {len(tot)} steps of ~{per_step:.1f} s, "
              f"full LM solves, {cores} worker processes")
    return done / el, iters / el, used, sample, el, [t[2] for t in tot]


def _pool_init():
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    sys.path[:0] = [REPO, os.path.join(REPO, "src")]


# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--problems", type=int, default=None, help="override the problem count")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="f64", choices=["mixed", "f64"])
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=16)
    ap.add_argument("--kernel", default="auto", help="solver kernel (LmParams.kernel)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    c = workload(args.config, args.problems)
    B = c["n_problems"]
    shape = f"{c['n_cams']} frames, K={c['K']:,}"
    cfg_json = {"workload": f"config{args.config}: batched {B:,} x ({shape})" if B > 1 else
                f"config{args.config}: {c['desc']}",
                "n_problems": B, "n_cams": c["n_cams"], "K": c["K"], "loss": c["loss"],
                "outlier_frac": c.get("outlier_frac", 0.0), "max_iters": c["max_iters"],
                "precision": args.precision, "kernel": args.kernel}
    dtype = "f64+f32" if args.precision == "mixed" else "f64"

    if args.impl == "reference":
        if rank != 0:
            return
        pps, ips, cores, sample, el, per = cpu_reference(c, args.cpu_budget, steps=args.steps,
                                                         warmup=args.warmup)
        line = {"metric": METRIC, "value": pps, "unit": "problems/s", "impl": "reference",
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * el / max(len(per), 1), "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic", "lm_iters_per_s": ips,
                "config": cfg_json,
                "cpu_baseline": {"value": pps, "unit": "problems/s", "cores": cores, "kind": "port",
                                 "sample": sample},
                "e2e": {"value": pps, "unit": "problems/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    import torch.distributed as dist
    from paper_2506_05558_b200 import dist as mdist
    from paper_2506_05558_b200 import solver

    # MBA_BENCH_ONE_GPU=1 (tests only): every rank on GPU 0 and the collectives
    # over gloo on host copies -- exercises the N-rank flow on a one-GPU box;
    # production runs use NCCL with one rank per GPU.
    one_gpu = os.environ.get("MBA_BENCH_ONE_GPU") == "1"
    dev_index = 0 if one_gpu else local
    torch.cuda.set_device(dev_index)
    coll = torch.device("cpu") if one_gpu else torch.device("cuda", dev_index)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lo, hi = mdist.shard_range(B, rank, world)
    t_gen = time.perf_counter()
    batch = make_shard(c, lo, hi - lo, workers=max(1, len(os.sched_getaffinity(0)) // max(world, 1)))
    hb = solver.pack_synth(batch)
    t_gen = time.perf_counter() - t_gen
    prm = solver.LmParams(max_iters=c["max_iters"], loss=c["loss"], precision=args.precision,
                          kernel=args.kernel)
    pinned = solver.pin(hb)
    db = solver.to_device(hb, pinned=pinned)
    # one step = solve this rank's shard + gather the complete outputs (R, t,
    # focal, points, statistics, status, traces) to rank 0 (dist.ShardedSolver)
    ss = mdist.ShardedSolver(db, prm, dist=dist, comm_device=coll)
    sol = ss.sol
    gather_bytes = ss.gather.bytes_per_step
    l2_bytes = 126 * 2 ** 20
    in_bytes = sum(v.numel() * v.element_size() for v in pinned.values() if v is not None)
    flush = None if in_bytes > l2_bytes else torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
    l2_note = ("inputs larger than L2 (%.2f GB per rank)" % (in_bytes / 1e9) if flush is None
               else "L2 flushed (256 MB write) between timed steps")

    def all_reduce(x, op):
        if world > 1:
            y = x.to(coll)
            dist.all_reduce(y, op=op)
            x.copy_(y)

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        ss.step()
    torch.cuda.synchronize()

    # ---------------- device-resident timed region ----------------
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    solve_ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev_index) as clk:
        for i in range(args.steps):
            if flush is not None:
                flush.fill_(i & 0xFF)
            starts[i].record(stream)
            solver.solve(db, prm, sol)
            solve_ends[i].record(stream)
            ss.gather.gather(sol)
            ends[i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [s_.elapsed_time(e) for s_, e in zip(starts, ends)]
    solve_ms = [s_.elapsed_time(e) for s_, e in zip(starts, solve_ends)]
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device="cuda")
    all_reduce(tot, dist.ReduceOp.MAX)
    total_ms = float(tot.item())

    n_iters = sol.n_iters.cpu().numpy()
    evals = sol.evals.cpu().numpy()
    status = sol.status.cpu().numpy()
    it_tot = torch.tensor([float(n_iters.sum())], dtype=torch.float64, device="cuda")
    all_reduce(it_tot, dist.ReduceOp.SUM)
    value = B * args.steps / (total_ms / 1e3)
    iters_per_s = float(it_tot.item()) * args.steps / (total_ms / 1e3)

    # roofline of the solve kernel on this rank (one mba_solve call per step),
    # timed by the events around the solve alone
    plan = solver.plan(db, prm)
    n_launch = solver.launches(db, prm)
    bytes_l, flops_l = algorithmic_work(batch, n_iters, evals, fused=plan > 0)
    mean_launch_s = statistics.mean(solve_ms) / 1e3
    peak, peak_kind = _peaks()
    achieved = bytes_l / mean_launch_s / 1e9
    # measured DRAM bytes of the solve kernel (ncu --set full capture, scaled per
    # problem; profiles/ncu_traffic.json) and its FP64/FP32 pipe utilisation
    traffic, ncu_pipe = None, None
    try:
        with open(os.path.join(REPO, "profiles", "ncu_traffic.json")) as fh:
            rec = json.load(fh).get(f"config{args.config}_{args.precision}")
        if rec:
            traffic = rec["dram_bytes_per_problem"] * (hi - lo)
            ncu_pipe = {k: rec[k] for k in ("fp64_pipe_frac", "fma_pipe_frac", "issue_active_frac", "source")
                        if k in rec}
    except (OSError, KeyError, ValueError):
        pass

    # ---------------- end to end through the public API ----------------
    # gsrecon.miniba.lm_solve_batch on this rank's shard as a list of
    # BaProblem objects (float64 uv, int64 indices, the reference's layout):
    # native walk + gather into pinned memory, H2D, device sort/pack, solve,
    # D2H, in-place write-back into the problems' arrays -- all inside the timed
    # call; the problems are reset to their initial values between calls.
    e2e = None
    if not args.no_e2e:
        del ss, sol
        torch.cuda.empty_cache()
        e2e = e2e_public_api(torch, dist, batch, c, args, world, coll, all_reduce)
        e2e["value"] = B * args.steps / e2e.pop("total_s")

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        pps, ips, cores, sample, el, _ = cpu_reference(c, args.cpu_budget)
        cpu = {"value": pps, "unit": "problems/s", "cores": cores, "kind": "port", "sample": sample,
               "lm_iters_per_s": ips}
    fp_peak = FP64_PEAK_TFLOPS if args.precision == "f64" else FP32_PEAK_TFLOPS
    fp_ach = flops_l / mean_launch_s / 1e12
    kname = (KERNEL_NAME if n_launch > 1 else KERNEL_NAME.split(" (")[0]) if plan > 0 else \
        "mba::solve_kernel family (plan %d)" % plan
    line = {
        "metric": METRIC, "value": value, "unit": "problems/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": dtype,
        "data": "synthetic", "config": cfg_json, "l2": l2_note, "lm_iters_per_s": iters_per_s,
        # the binding roofline of this on-chip kernel: the FP pipe (per-iteration
        # passes run out of shared memory; ncu DRAM traffic is inputs once + outputs)
        "roofline": {"bound": "fp64" if args.precision == "f64" else "fp32", "achieved": fp_ach,
                     "peak": fp_peak, "unit": "TFLOP/s", "frac": fp_ach / fp_peak, "traffic": traffic,
                     "kernel": kname, "plan": plan, "flops_per_launch": flops_l,
                     "peak_kind": "derived nominal 148 SM x %d lanes x 2 x 1.965 GHz" %
                                  (64 if args.precision == "f64" else 128),
                     "flops_model": "SURVEY 8d algorithmic flops of the executed iterations "
                                    "(reference trial counts)", "ncu": ncu_pipe},
        # the BASELINE metric's "% of HBM roofline": algorithmic pass bytes / launch time
        "roofline_hbm": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": bytes_l},
        "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": n_launch * args.steps,
        "clocks": clk.summary(),
        "gather": {"fields": "R, t, focal, points, final_stats, n_iters, status, costs, lambdas, "
                             "accepted, evals", "to": "rank 0", "in_timed_step": True,
                   "bytes_per_step": gather_bytes if world > 1 else 0},
        "solver": {"mean_lm_iters": float(n_iters.mean()), "mean_evals_per_iter":
                   float(evals.sum() / max(n_iters.sum(), 1)), "solve_ms_per_step": statistics.mean(solve_ms),
                   "status_counts": {str(k): int(v) for k, v in zip(*np.unique(status, return_counts=True))},
                   "gen_s": t_gen},
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def e2e_public_api(torch, dist, batch, c, args, world, coll, all_reduce):
    """Time gsrecon.miniba.lm_solve_batch host-to-host on this rank's shard."""
    from gsrecon.config import LmConfig
    from gsrecon.miniba import BaProblem, lm_solve_batch, _SOLVERS
    from paper_2506_05558_b200.batch import BatchSolver
    cam64 = batch.cam.astype(np.int64)
    pt64 = batch.pt.astype(np.int64)
    R0, t0, X0, f0 = batch.R.copy(), batch.t.copy(), batch.points.copy(), batch.focal.copy()
    probs = []
    for b in range(batch.n_problems):
        c0, c1 = batch.cam_off[b], batch.cam_off[b + 1]
        p0, p1 = batch.pt_off[b], batch.pt_off[b + 1]
        o0, o1 = batch.obs_off[b], batch.obs_off[b + 1]
        probs.append(BaProblem(R=batch.R[c0:c1], t=batch.t[c0:c1], focal=float(batch.focal[b]),
                               cx=float(batch.cx[b]), cy=float(batch.cy[b]), points=batch.points[p0:p1],
                               cam_idx=cam64[o0:o1], pt_idx=pt64[o0:o1], uv=batch.uv[o0:o1],
                               fixed_cams=batch.fixed[c0:c1], optimize_focal=batch.optimize_focal,
                               optimize_points=batch.optimize_points))
    bs = BatchSolver(None, n_chunks=args.e2e_chunks)
    _SOLVERS[torch.cuda.current_device()] = bs
    cfg = LmConfig(max_iters=c["max_iters"], loss=c["loss"], precision=args.precision)

    def reset():
        batch.R[...] = R0
        batch.t[...] = t0
        batch.points[...] = X0
        for p, f in zip(probs, f0):
            p.focal = float(f)

    for _ in range(args.warmup):
        reset()
        lm_solve_batch(probs, cfg)
    total = 0.0
    for _ in range(args.steps):
        reset()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t1 = time.perf_counter()
        infos = lm_solve_batch(probs, cfg)
        torch.cuda.synchronize()
        total += time.perf_counter() - t1
    tt = torch.tensor([total], dtype=torch.float64, device="cuda")
    all_reduce(tt, dist.ReduceOp.MAX)
    ok = int(np.sum(np.asarray(infos.status) >= 0))
    return {"total_s": float(tt.item()), "unit": "problems/s", "h2d_bytes_per_step": int(bs.h2d_bytes),
            "d2h_bytes_per_step": int(bs.d2h_bytes), "ms_per_step": 1e3 * float(tt.item()) / args.steps,
            "chunks": len(bs.chunks(batch.n_problems)) - 1, "host_threads": bs.threads,
            "gpu_launches_per_step": bs.launches, "problems_ok": ok,
            "path": "gsrecon.miniba.lm_solve_batch(list of BaProblem, float64 uv / int64 indices) -> "
                    "native gather -> pinned H2D -> mba_pack_obs -> mba_solve -> D2H -> in-place "
                    "write-back; host wall clock per call (perf_counter), max over ranks"}


if __name__ == "__main__":
    main()
