#!/usr/bin/env python
"""bench.py — batched gradient-based grasp search (Fast-Grasp'D hot path) on B200.

Metric (BASELINE.json): candidate-iterations/s (and grasps/s) at N GPUs.
Workload (BASELINE config 2, the largest single-GPU config the metric names):
  Allegro-style 4-finger hand (allegro16: J=16, N=2001 samples from the
  reference's sampler) grasping a 40 mm box and a cylinder (r 17.5 mm,
  h 70 mm), each an analytic SDF baked on a 64^3 FP32 grid over bounds +
  30 mm; 1024 candidates per GPU (512 per object), approach-sampled; the
  500-iteration optimizer schedule (dilation 0.02 -> 0, Adam lr 1e-3).
A step = one optimizer iteration of the whole batch: loss_gradient (7
perturbation sims x 8 Gauss-Seidel sweeps over every hand point, with the
adjoint) + Adam + apply_gradient_step for every candidate, i.e. 1024
candidate-iterations per GPU per step, two fused launches (one per object).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dgx|reference]

For N>1 run under torchrun: candidates are sharded across ranks (weak
scaling: 1024 per GPU), no collective in the timed loop; timing is the max
over ranks of the CUDA-event time. `--impl reference` times the reference's
own CPU implementation (oracle/_ref/libdgref.so: the unmodified reference
compiled from /root/reference with the grid SDF behind its contract) on the
host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ITERS = 500
CAND_PER_GPU = 1024
RES = 64
HAND = "allegro16"
# algorithmic FLOP per point-sweep: 160 backend-independent
# (50 forward + 110 adjoint) + 2 x F_sdf with F_sdf(grid trilinear + gradient + proxy) = 70
FLOP_PER_POINT_SWEEP = 160 + 2 * 70
# SURVEY §8(d) split by kernel: forward 50 + one grid query (70); adjoint 110 + one recompute (70)
FLOP_FWD_PER_POINT_SWEEP = 50 + 70
FLOP_ADJ_PER_POINT_SWEEP = 110 + 70
M_SIMS, GS = 7, 8


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dgx", choices=["dgx", "reference"])
    ap.add_argument("--candidates", type=int, default=CAND_PER_GPU)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def workload(rank: int, cand: int):
    from paper_2306_08132_b200 import init, model
    hand = model.HandDesc.asset(HAND)
    objs = [model.box_grid(res=RES), model.cylinder_grid(res=RES)]
    per = cand // len(objs)
    qs = [init.approach_init(o, hand, per, seed=17 + oi, first=rank * per) for oi, o in enumerate(objs)]
    return hand, objs, qs


def config_dict(cand: int, n_gpus: int) -> dict:
    return {
        "workload": f"config2: {HAND} (J=16, N=2001) on box 40mm + cylinder r17.5/h70mm SDF grids {RES}^3, "
                    f"{cand} candidates/GPU ({cand // 2}/object), {ITERS}-iteration schedule; step = 1 iteration",
        "hand": HAND, "candidates_per_gpu": cand, "objects": ["box40_grid64", "cylinder_grid64"],
        "sdf": f"fp32 trilinear grid {RES}^3, fp64 arithmetic", "iterations_schedule": ITERS,
        "perturbations": M_SIMS, "gs_iters": GS, "l2": "flushed between timed steps (256 MiB write)",
        "parallelism": f"candidates sharded over {n_gpus} GPU(s), no inner-loop collective",
    }


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons, sampled every 100 ms; only samples
    whose own timestamp falls inside the timed window are summarised."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(1.5)  # nvidia-smi start-up
        except OSError:
            self.proc = None
        return self

    def _read(self):
        import datetime
        for line in self.proc.stdout:
            c = [x.strip() for x in line.split(",")]
            try:
                ts = datetime.datetime.strptime(c[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                continue
            self.rows.append([ts] + c[1:])

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()
        time.sleep(0.3)  # let the last in-window sample arrive

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        win = [r for r in self.rows if len(r) >= 8 and self.t0 is not None and self.t0 - 0.05 <= r[0] <= self.t1 + 0.05]
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in win if num(r[1]) is not None]
        mx = [num(r[2]) for r in win if num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in win for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm), "window_s": (self.t1 - self.t0) if self.t0 else None}


def traffic_from_profiles():
    p = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get("dram_bytes_per_launch")
    return None


# ---------------------------------------------------------------------------
def cpu_reference_sample(hand_name, objs, qs, k, n_per_obj, threads, variant="glibc"):
    """Reference CPU path (oracle/_ref) on a bounded sample: n_per_obj candidates
    per object, one optimizer iteration at schedule index k. Returns
    (candidate-iterations, seconds)."""
    from oracle import ref
    rh = {"allegro16": lambda: ref.RefHand.load_xml(os.path.join(ROOT, "assets", "hands", "allegro16",
                                                                 "allegro16.xml"), 2000, 12345, variant=variant)}[
        hand_name]()
    done, secs = 0, 0.0
    for o, q in zip(objs, qs):
        ro = ref.RefObject.from_desc(o, variant=variant)
        sub = q[:n_per_obj]
        t0 = time.perf_counter()
        out = ref.optimize(ro, rh, sub, ref.default_params(), iters=ITERS, k_begin=k, k_end=k + 1, threads=threads)
        secs += time.perf_counter() - t0
        done += sub.shape[0]
        assert not np.any(out["status"]), "reference optimizer failed"
    return done, secs


def run_reference(args, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    hand, objs, qs = workload(0, args.candidates)
    n_per = max(1, min(qs[0].shape[0], 2 * threads))
    for w in range(args.warmup):
        cpu_reference_sample(HAND, objs, qs, w % ITERS, n_per, threads)
    done = secs = 0
    for s in range(args.steps):
        d, t = cpu_reference_sample(HAND, objs, qs, (args.warmup + s) % ITERS, n_per, threads)
        done += d
        secs += t
    v = done / secs
    sample = f"{n_per} candidates x 2 objects x 1 iteration per step, {threads} threads"
    print(json.dumps({
        "metric": "candidate-iterations/sec", "value": v, "unit": "candidate-iterations/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.candidates, args.gpus), "impl": "reference",
        "grasps_per_sec": v / ITERS,
        "cpu_baseline": {"value": v, "unit": "candidate-iterations/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": v, "unit": "candidate-iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
def run_dgx(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2306_08132_b200 import api, capi

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    hand_d, objs_d, qs = workload(rank, args.candidates)
    # one multi-object launch per step (dgx_optimize_multi): the two objects'
    # persistent launches overlap on side streams, so the second fills SMs as
    # the first drains
    ctx = api.Context(local_rank)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    hand = api.Hand(ctx, hand_d)
    objs = [api.GraspObject(ctx, o) for o in objs_d]
    proto, params, weights = api.StabilityProtocol.standard(), api.SimParams(), api.LossWeights()
    opt = api.OptConfig(iterations=ITERS)
    D = 6 + hand_d.num_joints
    counts = np.array([q.shape[0] for q in qs], np.int32)
    qall = np.concatenate(qs, axis=0)
    st = dict(q=torch.tensor(qall, device=dev), m=torch.zeros(qall.shape[0], D, dtype=torch.float64, device=dev),
              v=torch.zeros(qall.shape[0], D, dtype=torch.float64, device=dev),
              status=torch.zeros(qall.shape[0], dtype=torch.int32, device=dev))
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flags = capi.DGX_DEVICE_PTRS | capi.DGX_ASYNC

    def step(k, ev=None):
        k %= ITERS  # long runs wrap around the schedule (any iterate is a valid workload)
        if ev is not None:
            ev[0].record(stream)
        api.optimize_multi(ctx, objs, hand, st["q"], counts, proto, params, weights, opt, k_begin=k, k_end=k + 1,
                           adam_m=st["m"], adam_v=st["v"], flags=flags, status=st["status"])
        if ev is not None:
            ev[1].record(stream)

    clk = ClockSampler(local_rank).start()
    for w in range(args.warmup):
        step(w)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launches
    step_ms = []
    clk.mark_start()
    for s in range(args.steps):
        flush.zero_()  # L2 flush, outside the timed events
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        step(args.warmup + s, ev)
        torch.cuda.synchronize()
        step_ms.append(ev[0].elapsed_time(ev[1]))
    torch.cuda.synchronize()
    clk.mark_end()
    clk.stop()
    if world > 1:
        dist.barrier()
    launches = ctx.launches - launches0
    total_ms = sum(step_ms)
    status_bad = int(torch.count_nonzero(st["status"]))
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    cand_total = args.candidates * world
    value = cand_total * args.steps / (max_ms * 1e-3)

    # ---- end to end through the public host API (host arrays in / out, synchronous) ----
    # The step's inputs live in pinned host memory; the library copies them in,
    # runs the fused iteration and copies q / m / v / status / the iterate's
    # losses + gradient record back, every step.
    def pinned(a):
        t = torch.empty(a.shape, dtype=a.dtype, pin_memory=True)
        t.copy_(a)
        return t.numpy()

    host = dict(q=pinned(st["q"].cpu()), m=pinned(st["m"].cpu()), v=pinned(st["v"].cpu()))
    Bt = host["q"].shape[0]
    status_h = pinned(torch.zeros(Bt, dtype=torch.int32))
    traj_h = pinned(torch.zeros((Bt, 1, 3 + host["m"].shape[1]), dtype=torch.float64))
    ctx.set_stream(None)
    k0 = args.warmup + args.steps
    h2d = d2h = 0
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for s in range(args.steps):
        ks = (k0 + s) % ITERS
        out = api.optimize_multi(ctx, objs, hand, host["q"], counts, proto, params, weights, opt, k_begin=ks,
                                 k_end=ks + 1, adam_m=host["m"], adam_v=host["v"], record=True,
                                 status=status_h, traj=traj_h, inplace=True)
        nb = host["q"].nbytes + host["m"].nbytes + host["v"].nbytes
        h2d += nb + out["status"].nbytes
        d2h += nb + out["traj"].nbytes + out["status"].nbytes
    e2e_s = time.perf_counter() - t0
    t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_value = cand_total * args.steps / float(t.item())

    # ---- per-kernel launch durations (roofline of the dominant kernel) ----
    # One object's 512-candidate launches on one stream, CUDA events around
    # every launch on that stream (dgx_ctx_set_kernel_timing), L2 flushed
    # between steps; the same launches the ncu launch list shows serialised.
    ctx.set_stream(stream.cuda_stream)
    n0 = int(counts[0])
    sub = {k: st[k][:n0] for k in ("q", "m", "v", "status")}
    ktimes = None
    for phase in ("warm", "timed"):
        ctx.set_kernel_timing(phase == "timed")
        for s in range(3 if phase == "warm" else args.steps):
            flush.zero_()
            ks = (k0 + s) % ITERS
            api.optimize(ctx, objs[0], hand, sub["q"], proto, params, weights, opt, k_begin=ks, k_end=ks + 1,
                         adam_m=sub["m"], adam_v=sub["v"], status=sub["status"], flags=flags)
        torch.cuda.synchronize()
    ktimes = ctx.kernel_times()
    ctx.set_kernel_timing(False)

    if rank == 0:
        L = capi.load()
        import ctypes as C
        pk, pms = C.c_double(), C.c_double()
        capi.check(L.dgx_fp64_peak(local_rank, C.byref(pk), C.byref(pms)))
        n_pts = hand_d.num_samples
        flop_cand_iter = M_SIMS * GS * n_pts * FLOP_PER_POINT_SWEEP
        pts_sweeps = M_SIMS * GS * n_pts
        kern = {}
        for kind, per_ps in (("forward", FLOP_FWD_PER_POINT_SWEEP), ("adjoint", FLOP_ADJ_PER_POINT_SWEEP),
                             ("fused", FLOP_PER_POINT_SWEEP)):
            ms_tot, cnt = ktimes[kind]
            if cnt:
                ms = ms_tot / cnt
                kern[kind] = {"avg_launch_ms": ms, "launches": cnt, "candidates_per_launch": n0,
                              "flop_per_candidate_iteration": pts_sweeps * per_ps,
                              "achieved_tflops": pts_sweeps * per_ps * n0 / (ms * 1e-3) / 1e12}
        dom = max(kern, key=lambda k: kern[k]["avg_launch_ms"])
        step_kernel_ms = sum(v["avg_launch_ms"] for v in kern.values())
        for v in kern.values():
            v["share_of_serialised_step"] = v["avg_launch_ms"] / step_kernel_ms
        achieved = kern[dom]["achieved_tflops"]
        traffic = traffic_from_profiles()
        result = {
            "metric": "candidate-iterations/sec", "value": value, "unit": "candidate-iterations/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (approach-sampled configurations, analytic SDFs baked to grids)",
            "config": config_dict(args.candidates, world),
            "grasps_per_sec": value / ITERS,
            "e2e": {"value": e2e_value, "unit": "candidate-iterations/s",
                    "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
                    "path": "api.optimize_multi -> dgx_optimize_multi with pinned host arrays (q, adam m/v in; "
                            "q, m, v, status, iterate losses + gradient out), synchronous, wall clock"},
            "gpu_launches": launches,
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": pk.value, "unit": "TFLOP/s",
                         "frac": achieved / pk.value, "traffic": traffic, "kernel": dom,
                         "peak_source": "measured DFMA microbenchmark (dgx_fp64_peak, csrc/dgx_peak.cu)",
                         "flop_per_candidate_iteration": flop_cand_iter,
                         "timing": "dominant kernel: FLOP_alg of its half (SURVEY 8(d): adjoint 110 + 70 per "
                                   "point-sweep, forward 50 + 70) x candidates per launch / its mean launch "
                                   "duration, CUDA events on its stream, one object's launches, L2 flushed",
                         "kernels": kern,
                         "step_achieved_tflops": flop_cand_iter * args.candidates / (statistics.mean(step_ms) * 1e-3)
                         / 1e12,
                         "avg_step_ms": statistics.mean(step_ms)},
            "clocks": clk.summary(),
            "failed_candidates": status_bad,
        }
        if world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            hand_r, objs_r, qs_r = workload(0, args.candidates)
            n_per = max(1, min(qs_r[0].shape[0], 2 * threads))
            d, secs = cpu_reference_sample(HAND, objs_r, qs_r, 0, n_per, threads)
            result["cpu_baseline"] = {"value": d / secs, "unit": "candidate-iterations/s", "cores": threads,
                                      "kind": "reference",
                                      "sample": f"{n_per} candidates x 2 objects x 1 iteration (k=0), "
                                                f"{threads} std::threads, oracle/_ref/libdgref.so"}
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
    else:
        run_dgx(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
