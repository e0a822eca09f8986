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
    Sequential kernels: passes = 1 + n_eval, trials = n_eval. The cluster-resident
    kernel (fused=True) evaluates try 0 alone and tries 1..4 in one fused pass:
    passes = 1 + [n_eval >= 1] + [n_eval >= 2], trials = 1 or 5."""
    B = batch.n_problems
    K = np.diff(batch.obs_off).astype(np.float64)
    P = np.diff(batch.pt_off).astype(np.float64)
    live = np.arange(evals.shape[1])[None, :] < np.asarray(n_iters)[:, None]
    ev = evals.astype(np.float64) * live
    if fused:
        n_pass_sum = ((ev >= 1).astype(np.float64) + (ev >= 2)).sum(axis=1)
        n_eval_sum = np.where(ev >= 2, 5.0, ev).sum(axis=1)
    else:
        n_pass_sum = n_eval_sum = ev.sum(axis=1)
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


def cpu_reference(c, budget_s=15.0, seed=0):
    """Solve problems 0, 1, 2, ... of the workload on all host cores until the
    time budget is used. Returns (problems/s, iterations/s, cores, sample)."""
    import multiprocessing as mp
    cores = len(os.sched_getaffinity(0))
    if c["n_problems"] == 1 and c["K"] >= 100000:
        # one stress problem: a full 50-iteration CPU solve takes ~20 min, so
        # time the first 2 LM iterations on one core and scale to the solve
        _pool_init()
        sec, it = _cpu_solve((c, 0, seed, 2))
        ips = it / sec
        return (ips / c["max_iters"], ips, 1, f"first 2 LM iterations of the single problem, 1 core "
                f"({sec:.1f} s); problems/s = iterations/s / {c['max_iters']}", sec)
    ctx = mp.get_context("spawn")
    done = iters = 0
    t0 = time.perf_counter()
    with ctx.Pool(cores, initializer=_pool_init) as pool:
        nxt = 0
        pending = []
        while True:
            while len(pending) < 2 * cores and nxt < c["n_problems"] and time.perf_counter() - t0 < budget_s:
                pending.append(pool.apply_async(_cpu_solve, ((c, nxt, seed, c["max_iters"]),)))
                nxt += 1
            if not pending:
                break
            r = pending.pop(0).get()
            done += 1
            iters += r[1]
    el = time.perf_counter() - t0
    used = min(cores, max(done, 1))
    sample = f"first {done} problems of the workload, full LM solves, {cores} worker processes"
    return done / el, iters / el, used, sample, el


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
    ap.add_argument("--e2e-chunks", type=int, default=4)
    ap.add_argument("--kernel", default="auto", help="solver kernel (LmParams.kernel)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    c = workload(args.config, args.problems)
    cfg_json = {"workload": f"config{args.config}: {c['desc']}", "n_problems": c["n_problems"],
                "n_cams": c["n_cams"], "K": c["K"], "loss": c["loss"], "max_iters": c["max_iters"],
                "precision": args.precision, "kernel": args.kernel}

    if args.impl == "reference":
        if rank != 0:
            return
        pps, ips, cores, sample, el = cpu_reference(c, args.cpu_budget)
        line = {"metric": METRIC, "value": pps, "unit": "problems/s", "impl": "reference",
                "n_gpus": args.gpus, "steps": 1, "warmup": 0, "ms_per_step": el * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic", "lm_iters_per_s": ips, "config": cfg_json,
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

    # MBA_BENCH_ONE_GPU=1 (tests only): every rank on GPU 0 and the (tiny)
    # collectives over gloo on host copies -- exercises the N-rank flow on a
    # one-GPU box; production runs use NCCL with one rank per GPU.
    one_gpu = os.environ.get("MBA_BENCH_ONE_GPU") == "1"
    dev_index = 0 if one_gpu else local
    torch.cuda.set_device(dev_index)
    backend = "gloo" if one_gpu else "nccl"
    coll = "cpu" if one_gpu else "cuda"
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    B = c["n_problems"]
    lo, hi = mdist.shard_range(B, rank, world)
    t_gen = time.perf_counter()
    batch = make_shard(c, lo, hi - lo, workers=max(1, len(os.sched_getaffinity(0)) // max(world, 1)))
    hb = solver.pack_synth(batch)
    t_gen = time.perf_counter() - t_gen
    prm = solver.LmParams(max_iters=c["max_iters"], loss=c["loss"], precision=args.precision,
                          kernel=args.kernel)
    pinned = solver.pin(hb)
    db = solver.to_device(hb, pinned=pinned)
    sol = solver.Solution(db, prm.max_iters)
    l2_bytes = 126 * 2 ** 20
    in_bytes = sum(v.numel() * v.element_size() for v in pinned.values() if v is not None)
    flush = None if in_bytes > l2_bytes else torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda")
    cfg_json["l2"] = ("inputs larger than L2 (%.2f GB per rank)" % (in_bytes / 1e9) if flush is None
                      else "L2 flushed (256 MB write) between timed steps")
    rows = mdist.padded_rows(B, world)
    gbufs = [torch.empty((rows, mdist.SUMMARY_WIDTH), dtype=torch.float64, device=coll)
             for _ in range(world)]

    def gather_step():
        """final gather of the per-problem summaries (the only collective)"""
        if world == 1:
            return None
        local = mdist.pack_summary(torch, sol.final_stats, sol.n_iters, sol.status, rows, "cuda")
        return mdist.gather_summaries(torch, dist, local.to(coll), B, world, gbufs)

    def all_reduce(x, op):
        if world > 1:
            y = x.to(coll)
            dist.all_reduce(y, op=op)
            x.copy_(y)

    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        solver.solve(db, prm, sol)
        gather_step()
    torch.cuda.synchronize()

    # ---------------- device-resident timed region ----------------
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev_index) as clk:
        for i in range(args.steps):
            if flush is not None:
                flush.fill_(i & 0xFF)
            starts[i].record(stream)
            solver.solve(db, prm, sol)
            gather_step()
            ends[i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
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

    # roofline of the solve kernel on this rank (one launch = one step)
    plan = solver.plan(db, prm)
    n_launch = solver.launches(db, prm)
    bytes_l, flops_l = algorithmic_work(batch, n_iters, evals, fused=plan > 0)
    mean_launch_s = statistics.mean(step_ms) / 1e3
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

    # ---------------- end to end through the C ABI with host buffers --------
    # PipelinedSolver: pinned host inputs -> H2D (copy stream) -> mba_solve
    # (compute stream) -> D2H of the solution, chunked so copies overlap solves.
    e2e = None
    if not args.no_e2e:
        del db, sol
        torch.cuda.empty_cache()
        ps = solver.PipelinedSolver(hb, prm, n_chunks=args.e2e_chunks)
        for _ in range(args.warmup):
            ps.run()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e_s = torch.cuda.Event(enable_timing=True)
        e_e = torch.cuda.Event(enable_timing=True)
        e_s.record(ps.copy)
        for _ in range(args.steps):
            ps.run()
        ps.wait()
        e_e.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        e_ms = torch.tensor([e_s.elapsed_time(e_e)], dtype=torch.float64, device="cuda")
        all_reduce(e_ms, dist.ReduceOp.MAX)
        e2e = {"value": B * args.steps / (float(e_ms.item()) / 1e3), "unit": "problems/s",
               "h2d_bytes_per_step": int(ps.h2d_bytes), "d2h_bytes_per_step": int(ps.d2h_bytes),
               "ms_per_step": float(e_ms.item()) / args.steps, "chunks": len(ps.parts),
               "path": "PipelinedSolver -> mba_solve (C ABI), pinned host buffers"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        pps, ips, cores, sample, el = cpu_reference(c, args.cpu_budget)
        cpu = {"value": pps, "unit": "problems/s", "cores": cores, "kind": "port", "sample": sample,
               "lm_iters_per_s": ips}
    line = {
        "metric": METRIC, "value": value, "unit": "problems/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64+f32" if args.precision == "mixed" else "f64",
        "data": "synthetic", "config": cfg_json, "lm_iters_per_s": iters_per_s,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": (KERNEL_NAME if n_launch > 1 else KERNEL_NAME.split(" (")[0]) if plan > 0 else "mba::solve_kernel family (plan %d)" % plan,
                     "plan": plan, "algorithmic_bytes_per_launch": bytes_l,
                     "note": "per-iteration passes run out of shared memory; DRAM traffic (ncu) is "
                             "inputs once + outputs, so the HBM fraction is low by design and the "
                             "binding resource is the FP pipe / issue rate (roofline_fp below)"},
        "roofline_fp": {"achieved": flops_l / mean_launch_s / 1e12,
                        "peak": FP64_PEAK_TFLOPS if args.precision == "f64" else FP32_PEAK_TFLOPS,
                        "unit": "TFLOP/s",
                        "frac": flops_l / mean_launch_s / 1e12 /
                                (FP64_PEAK_TFLOPS if args.precision == "f64" else FP32_PEAK_TFLOPS),
                        "pipe": "fp64" if args.precision == "f64" else "fp32",
                        "peak_kind": "derived nominal 148 SM x %d lanes x 2 x 1.965 GHz" %
                                     (64 if args.precision == "f64" else 128),
                        "flops_model": "SURVEY 8d algorithmic flops of the executed iterations",
                        "ncu": ncu_pipe},
        "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": n_launch * args.steps,
        "clocks": clk.summary(),
        "solver": {"mean_lm_iters": float(n_iters.mean()), "mean_evals_per_iter":
                   float(evals.sum() / max(n_iters.sum(), 1)),
                   "status_counts": {str(k): int(v) for k, v in zip(*np.unique(status, return_counts=True))},
                   "gen_s": t_gen},
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
