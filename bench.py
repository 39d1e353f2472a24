#!/usr/bin/env python
"""bench.py — batched gradient-based grasp search (Fast-Grasp'D hot path) on B200.

Metric (BASELINE.json): candidate-iterations/s (and grasps/s) at N GPUs.
Headline workload (BASELINE config 3, the largest single-GPU configuration in
BASELINE.json's `configs`):
  Shadow-style 5-finger full-DOF hand (shadow22_dense: J=22, N=4093 surface
  samples from the reference's own sampler, HandModel::load_xml(shadow22.xml,
  4096)) grasping a procedural blob body baked on a 128^3 FP32 SDF grid;
  4096 candidates per GPU, approach-sampled; the 500-iteration optimizer
  schedule (dilation 0.02 -> 0, Adam lr 1e-3).
A step = one optimizer iteration of the whole batch: loss_gradient (7
perturbation sims x 8 Gauss-Seidel sweeps over every hand point, with the
adjoint) + Adam + apply_gradient_step for every candidate, i.e. 4096
candidate-iterations per GPU per step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dgx|reference]
                  [--workload config3|config2|config4]

Multi-GPU: under torchrun (WORLD_SIZE set) every rank runs its own candidate
shard (weak scaling, 4096 per GPU; config4: whole objects per rank, strong
scaling) with no collective in the timed loop; timing is the max over ranks of
the CUDA-event time; the final records (q, status, last iterate's losses) are
gathered to rank 0 once, after timing. Without WORLD_SIZE, `--gpus N > 1`
spawns N local ranks itself, or exits non-zero when fewer GPUs are visible.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libdgref.so: the unmodified reference compiled from
/root/reference, with the grid SDF behind its record_dilated contract) on the
host cores, rank 0 only, on a bounded candidate sample progressed through the
same iterates k as the GPU arm.
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
M_SIMS, GS = 7, 8
# algorithmic FLOP per point-sweep: 160 backend-independent
# (50 forward + 110 adjoint) + 2 x F_sdf with F_sdf(grid trilinear + gradient + proxy) = 70
FLOP_PER_POINT_SWEEP = 160 + 2 * 70
# SURVEY §8(d) split by kernel: forward 50 + one grid query (70); adjoint 110 + one recompute (70)
FLOP_FWD_PER_POINT_SWEEP = 50 + 70
FLOP_ADJ_PER_POINT_SWEEP = 110 + 70

WORKLOADS = {
    "config3": dict(hand="shadow22_dense", hand_xml=("shadow22", 4096), cand=4096, scaling="weak",
                    desc="config3: shadow22_dense (J=22, N=4093) on a procedural blob SDF grid 128^3 (seed 3), "
                         "{cand} candidates/GPU, 500-iteration schedule; step = 1 iteration"),
    "config2": dict(hand="allegro16", hand_xml=("allegro16", 2000), cand=1024, scaling="weak",
                    desc="config2: allegro16 (J=16, N=2001) on box 40mm + cylinder r17.5/h70mm SDF grids 64^3, "
                         "{cand} candidates/GPU (half per object), 500-iteration schedule; step = 1 iteration"),
    "config4": dict(hand="barrett3", hand_xml=None, cand=1024, scaling="strong",
                    desc="config4: barrett3 (J=9, N=1999) x 64 procedural blob objects (64^3 grids) x {cand} "
                         "candidates = 65536, object-major over the GPUs; step = 1 iteration"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="dgx", choices=["dgx", "reference"])
    ap.add_argument("--workload", default="config3", choices=sorted(WORKLOADS))
    ap.add_argument("--candidates", type=int, default=None, help="per GPU (per object for config4)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    a = ap.parse_args()
    if a.warmup < 3:
        ap.error("--warmup must be >= 3")
    if a.candidates is None:
        a.candidates = WORKLOADS[a.workload]["cand"]
    return a


def objects(name: str, rank: int = 0, world: int = 1):
    """[(object index, ObjectDesc)] this rank runs."""
    from paper_2306_08132_b200 import model, shard
    if name == "config3":
        return [(0, model.blob_grid(seed=3, res=128))]
    if name == "config2":
        return [(0, model.box_grid(res=64)), (1, model.cylinder_grid(res=64))]
    return [(o, model.blob_grid(seed=o, res=64)) for o, _, _ in shard.object_major(64, 1, world, rank)]


def workload(name: str, rank: int, world: int, cand: int):
    """hand, [ObjectDesc], [q per object] for this rank (global candidate ids)."""
    from paper_2306_08132_b200 import init, model
    w = WORKLOADS[name]
    hand = model.HandDesc.asset(w["hand"])
    objs = objects(name, rank, world)
    if name == "config4":
        qs = [init.approach_init(o, hand, cand, seed=100 + oi) for oi, o in objs]
    else:
        per = cand // len(objs)
        qs = [init.approach_init(o, hand, per, seed=17 + oi if name == "config2" else 3, first=rank * per)
              for oi, o in objs]
    return hand, [o for _, o in objs], qs


def config_dict(name: str, cand: int, n_gpus: int) -> dict:
    w = WORKLOADS[name]
    out = {"workload": w["desc"].format(cand=cand), "hand": w["hand"], "iterations_schedule": ITERS,
           "perturbations": M_SIMS, "gs_iters": GS, "sdf": "fp32 trilinear grid, fp64 arithmetic",
           "l2": "flushed between timed steps (256 MiB write)"}
    if name == "config4":
        out.update(objects=64, candidates_per_object=cand,
                   parallelism=f"objects sharded over {n_gpus} GPU(s) (object-major), no inner-loop collective")
    else:
        out.update(candidates_per_gpu=cand,
                   parallelism=f"candidates sharded over {n_gpus} GPU(s), no inner-loop collective")
    return out


def ref_hand(name: str):
    from oracle import ref
    w = WORKLOADS[name]
    if w["hand_xml"] is None:
        return ref.RefHand.barrett3(variant="glibc")
    base, budget = w["hand_xml"]
    return ref.RefHand.load_xml(os.path.join(ROOT, "assets", "hands", base, base + ".xml"), budget, 12345,
                                variant="glibc")


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


def traffic_from_profiles(name: str, kernel: str, candidates_per_launch: float):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed ncu --set full capture of THIS workload (profiles/
    roofline_traffic.json, keyed by workload and kernel kind), scaled from the
    captured launch's candidate count to this run's average launch; None when
    that capture does not exist."""
    p = os.path.join(ROOT, "profiles", "roofline_traffic.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as f:
        d = json.load(f).get(name, {}).get(kernel)
    if not d:
        return None, None
    per = d["dram_bytes_per_launch"] / d["candidates_per_launch"]
    return per * candidates_per_launch, d["source"]


# ---------------------------------------------------------------------------
class RefSample:
    """The reference's CPU path (oracle/_ref/libdgref.so, glibc: the reference
    exactly) over a fixed candidate sample whose optimizer state (q, Adam m/v)
    is carried from iterate to iterate, so iterate k here is the same workload
    the GPU arm runs at its step k."""

    def __init__(self, name, objs, qs, n_per_obj, m=None, v=None):
        from oracle import ref
        self.ref = ref
        self.rh = ref_hand(name)
        self.ros = [ref.RefObject.from_desc(o, variant="glibc") for o in objs]
        self.q = [np.array(q[:n_per_obj], np.float64) for q in qs]
        self.m = [None if m is None else np.array(x[:n_per_obj]) for x in (m or [None] * len(qs))]
        self.v = [None if v is None else np.array(x[:n_per_obj]) for x in (v or [None] * len(qs))]

    def iterate(self, k, threads):
        """One optimizer iterate k for every sampled candidate -> (candidate-iterations, seconds)."""
        done, secs = 0, 0.0
        for i, ro in enumerate(self.ros):
            t0 = time.perf_counter()
            out = self.ref.optimize(ro, self.rh, self.q[i], self.ref.default_params(), iters=ITERS, k_begin=k,
                                    k_end=k + 1, adam_m=self.m[i], adam_v=self.v[i], threads=threads)
            secs += time.perf_counter() - t0
            done += self.q[i].shape[0]
            ok = out["status"] == 0  # a failed candidate stays where it failed (as on the GPU)
            self.q[i][ok], self.m[i], self.v[i] = out["q"][ok], out["m"], out["v"]
        return done, secs


def run_reference(args, rank):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    hand, objs, qs = workload(args.workload, 0, 1, args.candidates)
    n_per = max(1, min(qs[0].shape[0], (8 * threads) // len(objs)))
    rs = RefSample(args.workload, objs, qs, n_per)
    for w in range(args.warmup):  # iterates 0..W-1, as the GPU arm's warm-up
        rs.iterate(w % ITERS, threads)
    done = secs = 0
    for s in range(args.steps):
        d, t = rs.iterate((args.warmup + s) % ITERS, threads)
        done += d
        secs += t
    v = done / secs
    sample = (f"{n_per} candidates x {len(objs)} object(s) x 1 iteration per step (min(B, 8 x nproc)), "
              f"state carried across steps so step s runs iterate k = warmup + s like the GPU arm; "
              f"{threads} std::threads, oracle/_ref/libdgref.so")
    print(json.dumps({
        "metric": "candidate-iterations/sec", "value": v, "unit": "candidate-iterations/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / args.steps,
        "higher_is_better": True, "scaling": WORKLOADS[args.workload]["scaling"], "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": config_dict(args.workload, args.candidates, args.gpus),
        "impl": "reference", "grasps_per_sec": v / ITERS,
        "cpu_baseline": {"value": v, "unit": "candidate-iterations/s", "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": v, "unit": "candidate-iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ---------------------------------------------------------------------------
def run_dgx(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2306_08132_b200 import api, capi, shard

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    hand_d, objs_d, qs = workload(args.workload, rank, world, args.candidates)
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
    B_local = qall.shape[0]
    st = dict(q=torch.tensor(qall, device=dev), m=torch.zeros(B_local, D, dtype=torch.float64, device=dev),
              v=torch.zeros(B_local, D, dtype=torch.float64, device=dev),
              status=torch.zeros(B_local, dtype=torch.int32, device=dev))
    torch.cuda.synchronize()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    flags = capi.DGX_DEVICE_PTRS | capi.DGX_ASYNC

    def step(k, ev=None):
        k %= ITERS  # long runs wrap around the schedule (any iterate is a valid workload)
        if ev is not None:
            ev[0].record(stream)
        if len(objs) == 1:
            api.optimize(ctx, objs[0], hand, st["q"], proto, params, weights, opt, k_begin=k, k_end=k + 1,
                         adam_m=st["m"], adam_v=st["v"], flags=flags, status=st["status"])
        else:  # objects' launches overlap on side streams (dgx_optimize_multi)
            api.optimize_multi(ctx, objs, hand, st["q"], counts, proto, params, weights, opt, k_begin=k,
                               k_end=k + 1, adam_m=st["m"], adam_v=st["v"], flags=flags, status=st["status"])
        if ev is not None:
            ev[1].record(stream)

    clk = ClockSampler(local_rank).start()
    for w in range(args.warmup):
        step(w)
    torch.cuda.synchronize()
    # the CPU baseline's sample starts from this state (iterate k = warmup), so
    # it runs the same iterates the timed GPU steps run
    snap = {k: st[k].cpu().numpy().copy() for k in ("q", "m", "v")}
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
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    cand_total = B_local * world if args.workload != "config4" else 64 * args.candidates
    value = cand_total * args.steps / (max_ms * 1e-3)

    # ---- end to end through the public host API (host arrays in / out, synchronous) ----
    # The step's inputs live in pinned host memory; the library copies them in,
    # runs the iteration and copies q / m / v / status / the iterate's losses +
    # gradient record back, every step.
    def pinned(a):
        t = torch.empty(a.shape, dtype=a.dtype, pin_memory=True)
        t.copy_(a)
        return t.numpy()

    host = dict(q=pinned(st["q"].cpu()), m=pinned(st["m"].cpu()), v=pinned(st["v"].cpu()))
    status_h = pinned(torch.zeros(B_local, dtype=torch.int32))
    traj_h = pinned(torch.zeros((B_local, 1, 3 + D), dtype=torch.float64))
    ctx.set_stream(None)
    k0 = args.warmup + args.steps
    h2d = d2h = 0
    # one untimed call first: the host path runs on the context's side stream,
    # whose scratch is allocated on first use
    api.optimize_multi(ctx, objs, hand, host["q"].copy(), counts, proto, params, weights, opt, k_begin=k0 % ITERS,
                       k_end=k0 % ITERS + 1, adam_m=host["m"].copy(), adam_v=host["v"].copy(), record=True)
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

    # ---- final records gathered once, after timing: q, status,
    # the last iterate's losses; candidate order, rank 0 ----
    rec = np.concatenate([host["q"], status_h[:, None].astype(np.float64), traj_h[:, 0, :3]], axis=1)
    if args.workload == "config4":
        olo, ohi = shard.shard_range(64, world, rank)
        full = shard.gather_rows(rec, 64 * args.candidates, world, rank) if world > 1 else rec
        gathered = None if full is None else full.shape[0]
    else:
        full = shard.gather_rows(rec, cand_total, world, rank)
        gathered = None if full is None else full.shape[0]
    failed = None if full is None else int(np.count_nonzero(full[:, 7 + hand_d.num_joints]))

    # ---- per-kernel launch durations (roofline of the dominant kernel) ----
    # The bench's own launches on one stream, CUDA events around every launch
    # on that stream (dgx_ctx_set_kernel_timing), L2 flushed between steps.
    ctx.set_stream(stream.cuda_stream)
    n0 = int(counts[0])
    sub = {k: st[k][:n0] for k in ("q", "m", "v", "status")}
    ksteps = max(3, min(args.steps, 10))
    for phase in ("warm", "timed"):
        ctx.set_kernel_timing(phase == "timed")
        for s in range(3 if phase == "warm" else ksteps):
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
                # a step's n0 candidates may be split over several launches (scratch
                # chunks): a launch processes n0 * steps / launches candidates on average
                ms = ms_tot / cnt
                per_launch = n0 * ksteps / cnt
                kern[kind] = {"avg_launch_ms": ms, "launches": cnt, "steps": ksteps,
                              "candidates_per_launch": per_launch,
                              "flop_per_candidate_iteration": pts_sweeps * per_ps,
                              "achieved_tflops": pts_sweeps * per_ps * per_launch / (ms * 1e-3) / 1e12}
        dom = max(kern, key=lambda k: kern[k]["avg_launch_ms"] * kern[k]["launches"])
        step_kernel_ms = sum(v["avg_launch_ms"] * v["launches"] for v in kern.values())
        for v in kern.values():
            v["share_of_serialised_step"] = v["avg_launch_ms"] * v["launches"] / step_kernel_ms
        achieved = kern[dom]["achieved_tflops"]
        traffic, traffic_src = traffic_from_profiles(args.workload, dom, kern[dom]["candidates_per_launch"])
        result = {
            "metric": "candidate-iterations/sec", "value": value, "unit": "candidate-iterations/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
            "higher_is_better": True, "scaling": WORKLOADS[args.workload]["scaling"], "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (approach-sampled configurations, procedural / analytic SDFs baked to grids)",
            "config": config_dict(args.workload, args.candidates, world),
            "grasps_per_sec": value / ITERS,
            "e2e": {"value": e2e_value, "unit": "candidate-iterations/s",
                    "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
                    "path": "api.optimize_multi -> dgx_optimize_multi with pinned host arrays (q, adam m/v in; "
                            "q, m, v, status, iterate losses + gradient out), synchronous, wall clock"},
            "gpu_launches": launches,
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": pk.value, "unit": "TFLOP/s",
                         "frac": achieved / pk.value, "traffic": traffic, "traffic_source": traffic_src,
                         "kernel": dom,
                         "peak_source": "builder-measured DFMA microbenchmark (dgx_fp64_peak, csrc/dgx_peak.cu) "
                                        "on this GPU; nominal B200 FP64 37.2 TFLOP/s",
                         "frac_of_nominal_fp64": achieved / 37.2,
                         "flop_per_candidate_iteration": flop_cand_iter,
                         "timing": "dominant kernel: FLOP_alg of its part (SURVEY 8(d): forward 50 + 70, adjoint "
                                   "110 + 70, fused 300 per point-sweep) x candidates per launch / its mean launch "
                                   "duration, CUDA events on its stream, L2 flushed",
                         "kernels": kern,
                         "step_achieved_tflops": flop_cand_iter * (cand_total / world) /
                         (statistics.mean(step_ms) * 1e-3) / 1e12,
                         "avg_step_ms": statistics.mean(step_ms)},
            "clocks": clk.summary(),
            "gather": {"rows": gathered, "failed_candidates": failed,
                       "how": "shard.gather_rows (NCCL all-gather when N > 1) of q | status | losses, after timing"},
        }
        if world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            n_per = max(1, min(n0, (8 * threads) // len(objs)))
            qsnap = np.split(snap["q"], np.cumsum(counts)[:-1])
            msnap = np.split(snap["m"], np.cumsum(counts)[:-1])
            vsnap = np.split(snap["v"], np.cumsum(counts)[:-1])
            rs = RefSample(args.workload, objs_d, qsnap, n_per, msnap, vsnap)
            done = secs = 0
            for j in range(3):  # iterates warmup .. warmup + 2 from the GPU arm's own state
                d, t_ = rs.iterate((args.warmup + j) % ITERS, threads)
                done += d
                secs += t_
            result["cpu_baseline"] = {"value": done / secs, "unit": "candidate-iterations/s", "cores": threads,
                                      "kind": "reference",
                                      "sample": f"{n_per} candidates x {len(objs)} object(s) x 3 iterations "
                                                f"(k = {args.warmup}..{args.warmup + 2}, from the GPU arm's state at "
                                                f"the start of its timed region), {threads} std::threads, "
                                                f"oracle/_ref/libdgref.so"}
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _spawned(local_rank, args, world, port):
    os.environ.update(RANK=str(local_rank), LOCAL_RANK=str(local_rank), WORLD_SIZE=str(world),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    run_dgx(args, local_rank, world, local_rank)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        run_dgx(args, rank, world, local_rank)
        return
    if args.gpus > 1:  # no launcher: spawn one rank per GPU here
        import socket
        import torch
        import torch.multiprocessing as mp
        have = torch.cuda.device_count()
        if have < args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} requested but {have} CUDA device(s) visible")
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        mp.spawn(_spawned, args=(args, args.gpus, port), nprocs=args.gpus, join=True)
        return
    run_dgx(args, 0, 1, 0)


if __name__ == "__main__":
    main()
