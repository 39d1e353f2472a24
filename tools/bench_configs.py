"""Measure BASELINE.json configs 1, 3, 4, 5 on one B200 (config 2 is bench.py's
headline). Writes one JSON record per line to stdout.

  config1_mesh  the same on the reference's own representation: the
           make_icosphere(0.025, 3) triangle mesh, GPU mesh backend vs the
           UNMODIFIED reference (real MeshSdf) on the CPU.
  config1  barrett3 on the analytic sphere (R 25 mm), 64 candidates, 200 iterations:
           FULL run on the GPU, grasps/s, plus the reference CPU full run on a
           16-candidate subset and a distribution comparison (final loss /
           contact count / penetration, KS test).
  config3  shadow22_dense (J=22, N=4093) on a 128^3 procedural-blob grid,
           4096 candidates: candidate-iterations/s over a few iterations.
  config4  barrett3 x 64 procedural blob objects (64^3) x 1024 candidates
           (65,536 candidates, object-major, dgx_optimize_multi).
  config5  sweep: 3 hands x SDF resolution {32,64,128,256}^3 x candidates
           {256, 1024, 4096, 16384} (1024 / 16384 at 256^3) (one GPU; multi-GPU runs shard candidates
           with no collective, so aggregate = per-GPU x N).

usage: python tools/bench_configs.py [config1 config3 config4 config5]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2306_08132_b200 import api, capi, init, model  # noqa: E402

DEV = torch.device("cuda", 0)
FLAGS = capi.DGX_DEVICE_PTRS | capi.DGX_ASYNC


def timed_opt(ctx, objs, hand, hd, qs, iters, k_begin, k_end, reps=1):
    """Device-resident multi-object optimize over [k_begin, k_end); CUDA-event time."""
    stream = torch.cuda.Stream(DEV)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    D = 6 + hd.num_joints
    counts = np.array([q.shape[0] for q in qs], np.int32)
    q = torch.tensor(np.concatenate(qs, 0), device=DEV)
    m = torch.zeros(q.shape[0], D, dtype=torch.float64, device=DEV)
    v = torch.zeros_like(m)
    status = torch.zeros(q.shape[0], dtype=torch.int32, device=DEV)
    proto, params, w = api.StabilityProtocol.standard(), api.SimParams(), api.LossWeights()
    opt = api.OptConfig(iterations=iters)
    # warm-up: the first iteration of the schedule
    api.optimize_multi(ctx, objs, hand, q, counts, proto, params, w, opt, k_begin=0, k_end=1, adam_m=m, adam_v=v,
                       flags=FLAGS, status=status)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    api.optimize_multi(ctx, objs, hand, q, counts, proto, params, w, opt, k_begin=k_begin, k_end=k_end, adam_m=m,
                       adam_v=v, flags=FLAGS, status=status)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    ctx.set_stream(None)
    return ms, q.cpu().numpy(), int(torch.count_nonzero(status))


def config1():
    from scipy.stats import ks_2samp
    from oracle import ref
    hd = model.HandDesc.asset("barrett3")
    od = model.sphere(0.025)
    ctx = api.Context(0)
    hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
    B, K = 64, 200
    q0 = init.approach_init(od, hd, B, seed=1)
    ms, qf, bad = timed_opt(ctx, [obj], hand, hd, [q0], K, 1, K)
    ci_s = B * (K - 1) / (ms * 1e-3)
    # reference CPU: full 200-iteration runs on a 16-candidate subset (glibc build = the reference)
    rh = ref.RefHand.barrett3(variant="glibc")
    ro = ref.RefObject.from_desc(od, variant="glibc")
    sub = 16
    t0 = time.perf_counter()
    r = ref.optimize(ro, rh, q0[:sub], ref.default_params(), iters=K)
    cpu_s = time.perf_counter() - t0
    proto = api.StabilityProtocol.standard()
    eg, sg, _ = api.evaluate_losses(ctx, obj, hand, qf, proto, api.SimParams())
    er, sr = [], []
    for b in range(sub):
        er.append(ref.evaluate_losses(ro, rh, r["q"][b], ref.default_params()))
        sr.append([ref.sim_forward(ro, rh, r["q"][b], m, ref.default_params())[1] for m in range(7)])
    er, sr = np.array(er), np.array(sr)
    return dict(config="config1", workload="barrett3 (N=1999) on analytic sphere R=25mm, 64 candidates, 200 iterations",
                gpu_candidate_iterations_per_s=ci_s, gpu_full_run_s=ms * 1e-3 * K / (K - 1),
                gpu_grasps_per_s=B / (ms * 1e-3 * K / (K - 1)), failed=bad,
                cpu_reference_candidate_iterations_per_s=sub * K / cpu_s, cpu_threads=os.cpu_count(),
                cpu_subset=sub,
                ks_final_stable_loss_p=float(ks_2samp(eg[:, 0], er[:, 0]).pvalue),
                ks_contacts_p=float(ks_2samp(sg[:, :, 0].sum(1), sr[:, :, 0].sum(1)).pvalue),
                ks_penetration_p=float(ks_2samp(sg[:, :, 3].max(1), sr[:, :, 3].max(1)).pvalue),
                mean_final_loss_gpu=float(eg[:, 0].mean()), mean_final_loss_ref=float(er[:, 0].mean()))


def config1_mesh():
    """Config 1's mesh cross-check: the paper's representation,
    make_icosphere(0.025, 3) (1280 faces) through the UNMODIFIED reference
    MeshSdf on the CPU vs the GPU mesh backend, same mesh (bit-identical
    vertices), same hand, same initial configurations."""
    from scipy.stats import ks_2samp
    from oracle import ref
    hd = model.HandDesc.asset("barrett3")
    od = model.mesh_object(*model.icosphere_mesh(0.025, 3))
    ctx = api.Context(0)
    hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
    B, K = 64, 200
    q0 = init.approach_init(od, hd, B, seed=1)
    ms, qf, bad = timed_opt(ctx, [obj], hand, hd, [q0], K, 1, K)
    ci_s = B * (K - 1) / (ms * 1e-3)
    # throughput at a full-GPU batch
    Bw = 2048
    qw = init.approach_init(od, hd, Bw, seed=2)
    msw, _, badw = timed_opt(ctx, [obj], hand, hd, [qw], 500, 1, 3)
    rh = ref.RefHand.barrett3(variant="glibc")
    ro = ref.RefObject.icosphere(0.025, 3, variant="glibc")
    sub = 16
    t0 = time.perf_counter()
    r = ref.optimize(ro, rh, q0[:sub], ref.default_params(), iters=K)
    cpu_s = time.perf_counter() - t0
    proto = api.StabilityProtocol.standard()
    eg, sg, _ = api.evaluate_losses(ctx, obj, hand, qf, proto, api.SimParams())
    er, sr = [], []
    for b in range(sub):
        er.append(ref.evaluate_losses(ro, rh, r["q"][b], ref.default_params()))
        sr.append([ref.sim_forward(ro, rh, r["q"][b], m, ref.default_params())[1] for m in range(7)])
    er, sr = np.array(er), np.array(sr)
    return dict(config="config1_mesh",
                workload="barrett3 (N=1999) on make_icosphere(0.025, 3) mesh (1280 faces, alpha_phong 0.75), "
                         "64 candidates, 200 iterations",
                gpu_candidate_iterations_per_s=ci_s, gpu_full_run_s=ms * 1e-3 * K / (K - 1),
                gpu_grasps_per_s=B / (ms * 1e-3 * K / (K - 1)), failed=bad,
                gpu_candidate_iterations_per_s_B2048=Bw * 2 / (msw * 1e-3), failed_B2048=badw,
                cpu_reference_candidate_iterations_per_s=sub * K / cpu_s, cpu_threads=os.cpu_count(),
                cpu_subset=sub, cpu_reference="unmodified reference (glibc libm, real MeshSdf)",
                ks_final_stable_loss_p=float(ks_2samp(eg[:, 0], er[:, 0]).pvalue),
                ks_contacts_p=float(ks_2samp(sg[:, :, 0].sum(1), sr[:, :, 0].sum(1)).pvalue),
                ks_penetration_p=float(ks_2samp(sg[:, :, 3].max(1), sr[:, :, 3].max(1)).pvalue),
                mean_final_loss_gpu=float(eg[:, 0].mean()), mean_final_loss_ref=float(er[:, 0].mean()))


def scene_drop():
    """§8(f)-4 batched scene drop: scene-steps/s of step_on_table (sim.cpp:14-94)
    on the GPU (one warp per scene) vs the reference's own step_on_table on all
    host threads (oracle dgr_drop per scene, ctypes releases the GIL)."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import ref
    from paper_2306_08132_b200 import pipeline
    rows = []
    meshes = {"box (8 vertices)": lambda: ref.RefObject.box_mesh(0.04, 0.05, 0.03, variant="glibc"),
              "cylinder32 (66 vertices)": lambda: ref.RefObject.cylinder_mesh(0.0175, 0.07, 32, variant="glibc"),
              "icosphere3 (642 vertices)": lambda: ref.RefObject.icosphere(0.025, 3, variant="glibc"),
              "blob3 (642 vertices)": lambda: ref.RefObject.blob_mesh(0.021, 3, 0.5, 7, variant="glibc")}
    ctx = api.Context(0)
    stream = torch.cuda.Stream(DEV)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    for name, mk in meshes.items():
        ro = mk()
        V, F, _ = ro.mesh_export()
        od = model.mesh_object(V, F)
        obj = api.GraspObject(ctx, od)
        S, K = 8192, 2000
        s0 = torch.tensor(pipeline.scene_states(od, np.arange(S)), device=DEV)
        prm = api.DropParams(max_steps=K)
        api.drop(ctx, obj, s0[:256], prm)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        r = api.drop(ctx, obj, s0, prm)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        gsteps = float(r["steps"].sum().item())
        # reference CPU on a subset, all host threads
        sub = 64
        s0h = s0[:sub].cpu().numpy()
        t0 = time.perf_counter()
        with ThreadPoolExecutor(os.cpu_count()) as ex:
            res = list(ex.map(lambda b: ref.drop(ro, s0h[b], max_steps=K), range(sub)))
        cpu_s = time.perf_counter() - t0
        csteps = sum(x[1] for x in res)
        rows.append(dict(mesh=name, scenes=S, max_steps=K, gpu_ms=ms, gpu_scene_steps_per_s=gsteps / (ms * 1e-3),
                         gpu_scenes_per_s=S / (ms * 1e-3), mean_steps=gsteps / S,
                         at_rest_frac=float((r["steps"] < K).float().mean().item()),
                         cpu_reference_scene_steps_per_s=csteps / cpu_s, cpu_threads=os.cpu_count(), cpu_subset=sub))
    ctx.set_stream(None)
    return dict(config="scene_drop", workload="batched table drop, step_on_table until settled (100 calm steps) "
                                              "or 2 s; 8192 random-orientation scenes per mesh", rows=rows)


def metrics_sweep():
    """§8(f)-3: synthesis + grasp metrics. 256 barrett3 candidates on a 40 mm
    box MESH, 200 iterations on the GPU; contact generation at 1..10 mm
    (dgx_contacts_batch, one launch) and epsilon / GWS volume (host Qhull) for
    the initial and final grasps (SPEC ACCEPTANCE 5-6 shape)."""
    from paper_2306_08132_b200 import metrics
    hd = model.HandDesc.asset("barrett3")
    od = model.mesh_object(*model.box_mesh((0.04, 0.04, 0.04)))
    ctx = api.Context(0)
    hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
    B, K = 256, 200
    q0 = init.approach_init(od, hd, B, seed=21)
    ms, qf, bad = timed_opt(ctx, [obj], hand, hd, [q0], K, 1, K)
    thr = tuple(float(t) for t in range(1, 11))
    metrics.contacts(ctx, hand, obj, qf, thr)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        metrics.contacts(ctx, hand, obj, qf, thr)
    t_con = (time.perf_counter() - t0) / 5
    t0 = time.perf_counter()
    rep0 = metrics.evaluate(ctx, hand, obj, q0, thr, hull_thresholds_mm=(2.0, 5.0, 10.0))
    repf = metrics.evaluate(ctx, hand, obj, qf, thr, hull_thresholds_mm=(2.0, 5.0, 10.0))
    t_eval = (time.perf_counter() - t0) / 2
    s0, sf = metrics.threshold_sweep(rep0), metrics.threshold_sweep(repf)
    top = metrics.top_k(repf, 10, threshold_index=4)
    c5_0 = np.array([r[4]["contacts"] for r in rep0])
    c5_f = np.array([r[4]["contacts"] for r in repf])
    e5_f = np.array([r[4]["epsilon"] for r in repf])
    return dict(config="metrics_sweep", workload="barrett3 on a 40 mm box mesh, 256 candidates x 200 iterations; "
                                                 "metrics at 1..10 mm", opt_s=ms * 1e-3, failed=bad,
                contacts_kernel_grasps_per_s_10_thresholds=B / t_con,
                evaluate_s_per_grasp_hulls_at_3_thresholds=t_eval / B, hull_max_contacts=32,
                frac_more_contacts_at_5mm=float(np.mean(c5_f > c5_0)), frac_eps_positive_at_5mm=float(np.mean(e5_f > 0)),
                sweep_init=s0, sweep_final=sf,
                top10_mean_eps_5mm=float(np.mean([repf[i][4]["epsilon"] for i in top])),
                top10_mean_CA_cm2_5mm=float(np.mean([repf[i][4]["contact_area_cm2"] for i in top])))


def acceptance5():
    """SPEC ACCEPTANCE 5 on the GPU path: 20 seeds x 3 desk-scale MESH objects
    (cube, cylinder, blob) with the 3-finger hand, 200 iterations. Fraction of
    runs ending with (a) more 5 mm contacts than the initialization, (b)
    L_stable reduced >= 50%, (c) epsilon > 0 at 5 mm; the spec asks >= 70%."""
    from oracle import ref
    from paper_2306_08132_b200 import metrics
    hd = model.HandDesc.asset("barrett3")
    ctx = api.Context(0)
    hand = api.Hand(ctx, hd)
    objs = {"cube40": model.mesh_object(*model.box_mesh((0.04, 0.04, 0.04))),
            "cylinder": model.mesh_object(*ref.RefObject.cylinder_mesh(0.0175, 0.07, 32).mesh_export()[:2]),
            "blob": model.mesh_object(*ref.RefObject.blob_mesh(0.021, 3, 0.5, 7).mesh_export()[:2])}
    rows = []
    proto, params = api.StabilityProtocol.standard(), api.SimParams()
    for name, od in objs.items():
        obj = api.GraspObject(ctx, od)
        B, K = 20, 200
        q0 = init.approach_init(od, hd, B, seed=5)
        ms, qf, bad = timed_opt(ctx, [obj], hand, hd, [q0], K, 1, K)
        l0, _, _ = api.evaluate_losses(ctx, obj, hand, q0, proto, params)
        lf, _, _ = api.evaluate_losses(ctx, obj, hand, qf, proto, params)
        r0 = metrics.evaluate(ctx, hand, obj, q0, (5.0,))
        rf = metrics.evaluate(ctx, hand, obj, qf, (5.0,))
        a = np.array([rf[b][0]["contacts"] > r0[b][0]["contacts"] for b in range(B)])
        bb = lf[:, 0] <= 0.5 * l0[:, 0]
        c = np.array([rf[b][0]["epsilon"] > 0 for b in range(B)])
        rows.append(dict(object=name, runs=B, more_contacts=float(a.mean()), stable_halved=float(bb.mean()),
                         eps_positive=float(c.mean()), all_three=float((a & bb & c).mean()),
                         mean_stable_init=float(l0[:, 0].mean()), mean_stable_final=float(lf[:, 0].mean()),
                         gpu_s=ms * 1e-3, failed=bad))
    return dict(config="acceptance5", workload="barrett3, 20 seeds x {cube, cylinder, blob} meshes, 200 iterations",
                rows=rows)


def mesh_scaling():
    """SPEC ACCEPTANCE 7's BVH check on the GPU mesh backend: per-iteration
    cost vs face count (icospheres of 1280 / 5120 / 20480 faces, barrett3,
    2048 candidates)."""
    hd = model.HandDesc.asset("barrett3")
    ctx = api.Context(0)
    hand = api.Hand(ctx, hd)
    rows = []
    for sub in (3, 4, 5):
        V, F = model.icosphere_mesh(0.025, sub)
        od = model.mesh_object(V, F)
        obj = api.GraspObject(ctx, od)
        B = 2048
        q0 = init.approach_init(od, hd, B, seed=1)
        ms, _, bad = timed_opt(ctx, [obj], hand, hd, [q0], 500, 1, 3)
        rows.append(dict(faces=int(F.shape[0]), cand_iter_per_s=B * 2 / (ms * 1e-3), ms_per_iteration=ms / 2,
                         failed=bad))
    return dict(config="mesh_scaling", workload="barrett3 on icosphere meshes, 2048 candidates, 2 iterations",
                rows=rows)


def config3():
    hd = model.HandDesc.asset("shadow22_dense")
    od = model.blob_grid(seed=3, res=128)
    ctx = api.Context(0)
    hand, obj = api.Hand(ctx, hd), api.GraspObject(ctx, od)
    B, K = 4096, 500
    q0 = init.approach_init(od, hd, B, seed=3)
    ms, _, bad = timed_opt(ctx, [obj], hand, hd, [q0], K, 1, 4)
    return dict(config="config3", workload="shadow22_dense (J=22, N=4093) on 128^3 procedural blob grid, 4096 candidates",
                gpu_candidate_iterations_per_s=B * 3 / (ms * 1e-3), failed=bad, iterations_timed="1..3 of 500")


def config4():
    hd = model.HandDesc.asset("barrett3")
    ods = [model.blob_grid(seed=s, res=64) for s in range(64)]
    ctx = api.Context(0)
    hand = api.Hand(ctx, hd)
    objs = [api.GraspObject(ctx, o) for o in ods]
    per = 1024
    qs = [init.approach_init(o, hd, per, seed=100 + i) for i, o in enumerate(ods)]
    ms, _, bad = timed_opt(ctx, objs, hand, hd, qs, 500, 1, 3)
    return dict(config="config4", workload="barrett3 x 64 procedural blob objects (64^3) x 1024 candidates = 65536",
                gpu_candidate_iterations_per_s=64 * per * 2 / (ms * 1e-3), failed=bad, iterations_timed="1..2 of 500")


def config5():
    out = []
    ctx = api.Context(0)
    for hname in ("barrett3", "allegro16", "shadow22"):
        hd = model.HandDesc.asset(hname)
        hand = api.Hand(ctx, hd)
        for res in (32, 64, 128, 256):
            od = model.blob_grid(seed=11, res=res)
            obj = api.GraspObject(ctx, od)
            for B in ((256, 1024, 4096, 16384) if res < 256 else (1024, 16384)):
                q0 = init.approach_init(od, hd, B, seed=5)
                ms, _, bad = timed_opt(ctx, [obj], hand, hd, [q0], 500, 1, 2)
                out.append(dict(hand=hname, sdf_res=res, candidates=B, cand_iter_per_s=B / (ms * 1e-3), failed=bad))
    return dict(config="config5", workload="sweep: hands x SDF resolution x candidates (1 GPU)", rows=out)


def main():
    which = sys.argv[1:] or ["config1", "config1_mesh", "config3", "config4", "config5", "scene_drop", "metrics_sweep",
                                 "mesh_scaling"]
    for w in which:
        t = time.time()
        rec = globals()[w]()
        rec["wall_s"] = time.time() - t
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
