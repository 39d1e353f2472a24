// dgx_lane_adj.cuh — the split adjoint with one THREAD per (candidate, sim).
// Included by dgx_kernels.cu inside namespace dgx (uses its device helpers).
//
// The CTA adjoint (kernel_body<Sdf, kPhaseAdj>) gives each perturbation sim a
// warp and parallelises the leak recurrence over lanes: every block of 32 S
// positions is staged, composed into per-lane 3x3 affine maps, scanned across
// lanes (Kogge-Stone) and re-walked. That parallel prefix costs more than the
// recurrence itself (ncu, config 3: ~560 thread-instructions per point-sweep,
// 7 warps / SM at 255 registers, FP64 pipe 28%).
//
// Here a thread walks its sim's whole reverse sweep serially, exactly in the
// reference tape's order (tape.cpp:27-114): per position, the leak geometry of
// the frozen state (sim.hpp:105-125; the same leak_geo / leak_coef as the CTA
// adjoint), then adj_x <- adj_x - s n and the point adjoint folded into the
// per-link force / torque sums. No map composition, no scan and no shuffles.
// The 32 lanes of a warp are 32 (candidate, sim) tasks walking the
// SAME position sequence (sweep * N + i, descending) in lockstep, so the point
// index, its link and the link-change flushes are warp-uniform; only a lane's
// logged corrections (its run boundaries) diverge. U positions are processed
// per step: their geometry is independent (issued together: ILP), the
// recurrence then applies them in order. The warp's candidates' points are
// staged per block of positions in shared memory (cp.async, double-buffered).
//
// Logged corrections and frictions are reversed with the same closed forms as
// the CTA adjoint (correction_linear, friction_adj; dgx_adjoint.cuh), one
// thread each. Per-link sums go to task_ft transposed ([6L][tasks]: the
// warp-uniform flushes are coalesced). lane_epi_kernel then runs each
// candidate's epilogue (candidate_epilogue: sim-order reductions, FK adjoint,
// Adam, step) with one warp per candidate.
//
// Parity: forward values are untouched (the forward kernel is unchanged);
// gradients follow the tape's sequential order and match it to rounding
// (tests/test_gpu_parity.py bars), as the CTA adjoint does.
#pragma once

constexpr int kLaneAdjThreads = 32;  // one warp per CTA: tasks spread over all SMs' schedulers
constexpr int kEpiWarps = 4;
// min resident 1-warp CTAs per SM the register budget is sized for (1: up to
// 255 registers; A/B knob)
#ifndef DGX_LANE_MINB
#define DGX_LANE_MINB 1
#endif
// staged block of positions (a multiple of kLaneU: windows never straddle blocks)
#ifndef DGX_LANE_BLK
#define DGX_LANE_BLK 32
#endif
constexpr int kLaneBlk = DGX_LANE_BLK;
static_assert(kLaneAdjThreads == 32 && kLaneBlk % kLaneU == 0, "lane adjoint: one warp per CTA, windows tile the blocks");
// staged points: per buffer and candidate of the warp a row of x / y / z for
// kLaneBlk positions; rows 3 kLaneBlk + 2 doubles apart (with 32: 196 words,
// so the warp's <= 6 candidates (M = 7) fall on distinct banks)
constexpr int kLaneRowArr = kLaneBlk, kLaneRow = 3 * kLaneRowArr + 2;
__host__ __device__ inline int lane_cands_per_warp(int M) { return (31 / M + 2) < 32 ? (31 / M + 2) : 32; }
__host__ __device__ inline int lane_smem_bytes(int M) { return 2 * lane_cands_per_warp(M) * kLaneRow * 8; }
#ifndef DGX_LANE_CELL_NOL1
#define DGX_LANE_CELL_NOL1 0
#endif
// cell loads: 0 plain (L1 reuse between consecutive points: no_allocate measured
// 35.9 vs 30.9 ms), 1 L1::no_allocate, 2 L1::evict_first
constexpr int kLaneCellNoL1 = DGX_LANE_CELL_NOL1;
// grids: grid_finish_uniform (one normalisation, branch-free outside handling)
#ifndef DGX_LANE_UNIFORM_FINISH
#define DGX_LANE_UNIFORM_FINISH 1
#endif
// point staging copies with an L2 evict-first policy
// the R-node adjoint accumulated in the world frame (sum rel (x) n s), mapped back at corrections
#ifndef DGX_LANE_ARW
#define DGX_LANE_ARW 1
#endif
#ifndef DGX_LANE_FMA_U
#define DGX_LANE_FMA_U 1
#endif
#ifndef DGX_LANE_RAW_GEO
#define DGX_LANE_RAW_GEO 1
#endif
#ifndef DGX_LANE_PTS_FK
#define DGX_LANE_PTS_FK 0
#endif
#ifndef DGX_LANE_PTS_EVICT_FIRST
#define DGX_LANE_PTS_EVICT_FIRST 1
#endif

// Geometry prefetch split: grids issue their cell loads for all U positions
// before finishing any (grid_fetch / grid_finish); other backends classify in
// one go.
template <class Sdf>
struct GeoPre {
  __device__ __forceinline__ void fetch(const Sdf&, V3) {}
  __device__ __forceinline__ FastEval finish(const Sdf& s, V3 r, double radius) const { return classify(s, r, radius); }
  __device__ __forceinline__ RawEval finish_raw(const Sdf& s, V3 r, double radius) const {
    const FastEval fe = classify(s, r, radius);
    return RawEval{fe.cls, fe.g, fdot(fe.g, fe.g)};
  }
};
template <>
struct GeoPre<GridSdf> {
  GridFetch f;
  __device__ __forceinline__ void fetch(const GridSdf& s, V3 r) { grid_fetch<kLaneCellNoL1, DGX_LANE_FMA_U != 0>(s, r, f); }
  __device__ __forceinline__ FastEval finish(const GridSdf& s, V3 r, double radius) const {
#if DGX_LANE_UNIFORM_FINISH
    return grid_finish_uniform(s, r, f, radius);
#else
    return grid_finish(s, r, f, radius);
#endif
  }
  __device__ __forceinline__ RawEval finish_raw(const GridSdf& s, V3 r, double radius) const {
    return grid_finish_raw(s, r, f, radius);
  }
};

// Per-thread link accumulator: F_l = sum a_p, T_l = sum p x a_p over the
// current link, added into the task's transposed row on a link change.
struct LaneFt {
  int link = -1;
  V3 F{0.0, 0.0, 0.0}, T{0.0, 0.0, 0.0};
  __device__ __forceinline__ void flush(double* ftT, size_t nt) {
    if (link < 0) return;
    double* d = ftT + static_cast<size_t>(6 * link) * nt;
    d[0] += F.x; d[nt] += F.y; d[2 * nt] += F.z;
    d[3 * nt] += T.x; d[4 * nt] += T.y; d[5 * nt] += T.z;
    link = -1;
    F = V3{0.0, 0.0, 0.0};
    T = V3{0.0, 0.0, 0.0};
  }
  __device__ __forceinline__ void add(double* ftT, size_t nt, int l, V3 ap, V3 p) {
    DGX_ASSERT(l >= 0 && l < 32);
    if (l != link) {
      flush(ftT, nt);
      link = l;
    }
    F = F + ap;
    T = T + fcross(p, ap);
  }
};

// Where a position's world point comes from: the warp's staged block
// (StagedPts) or, with DGX_LANE_PTS_FK, rebuilt from the hand's sample and the
// candidate's link transform (FkPts: p = R_l s + t_l, the forward's own FK
// expression, so the same bits; s and the link are warp-uniform, the link
// transform is reloaded only when the walk changes link).
struct StagedPts {
  const double* ps;  // this lane's candidate row of the current block
  int top;           // position of the row's entry 0
  __device__ __forceinline__ V3 get(int pos, int) const {
    const int j = top - pos;
    DGX_ASSERT(j >= 0 && j < kLaneRowArr);
    return V3{ps[j], ps[kLaneRowArr + j], ps[2 * kLaneRowArr + j]};
  }
};
struct FkPts {
  const double* samples;
  const int* sample_link;
  const double* links;  // the candidate's link transforms [L][12] (R row-major, t)
  int cl = -1;
  M3 R;
  V3 tr;
  __device__ __forceinline__ V3 get(int, int i) {
    const int l = sample_link[i];
    if (l != cl) {
#pragma unroll
      for (int m = 0; m < 9; ++m) R.m[m] = links[12 * l + m];
      tr = V3{links[12 * l + 9], links[12 * l + 10], links[12 * l + 11]};
      cl = l;
    }
    const V3 sp{samples[3 * i], samples[3 * i + 1], samples[3 * i + 2]};
    return mul(R, sp) + tr;
  }
};

// The leak steps of U consecutive descending positions pos, pos-1, ... (point
// indices i, i-1, ... wrapping at N) with the frozen state (xk, Rk); slot u
// takes part iff pos - u > lim (above the lane's next correction). The points
// come from the warp's staged block (ps: this lane's candidate row, x / y / z
// at ps[0 / kLaneRowArr / 2 kLaneRowArr + j], j = jb + u).
template <int U, class Sdf, class Pts>
__device__ __forceinline__ void lane_leak_steps(const Sdf& sdf, const SimEnv& e, int pos, int i, int lim, V3 xk,
                                                const M3& Rk, V3 G, V3& a, M3& aR, LaneFt& acc, double* ftT,
                                                size_t nt, Pts& pts) {
  V3 p[U], rel[U], rl[U];
  int ii[U];
  GeoPre<Sdf> pre[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    ii[u] = i - u < 0 ? i - u + e.N : i - u;
    DGX_ASSERT(ii[u] >= 0 && ii[u] < e.N);
    p[u] = pts.get(pos - u, ii[u]);
    rel[u] = p[u] - xk;
    rl[u] = ftmul_add(Rk, rel[u], e.O->com);
    pre[u].fetch(sdf, rl[u]);
  }
  double c1[U], c0[U];
  V3 n[U];
#if !(DGX_LANE_ARW && DGX_LANE_RAW_GEO)
  V3 g[U];  // the local-frame gradient (the emission's R-node term in the local frame)
#endif
  bool on[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
#if DGX_LANE_RAW_GEO
    // the leak coefficients from the unnormalised direction v (|v|^2 = v2):
    // w = inv_mass + aa.Iw aa with aa = rel x n, n = R v / |v|, so
    // v2 w = inv_mass v2 + av.Iw av with av = rel x R v; the normalisation
    // (rsqrt) runs beside that chain instead of in front of it
    const RawEval fr = pre[u].finish_raw(sdf, rl[u], e.radius);
    double sg = 1.0;
    V3 v = fr.v;
    double v2 = fr.v2;
    on[u] = pos - u > lim && fr.cls > 0;
    if (pos - u > lim && fr.cls == 0) {  // near the decision boundary: the exact (bit-exact) query decides
      PointEval pe;
      eval_point(sdf, e, ii[u], xk, Rk, true, pe);
      on[u] = !(pe.rho_d < 0.0);
      if (on[u]) {
        v = pe.q.grad;
        v2 = fdot(v, v);
        sg = pe.fb ? static_cast<double>(pe.q.sign) : 1.0;
      }
    }
    const V3 nv = fmul(Rk, v);
    const V3 av = fcross(rel[u], nv);
    const V3 Iav = fmul(e.O->Iw, av);
    const double den = fma(e.O->inv_mass, v2, fdot(av, Iav));  // v2 w
    on[u] = on[u] && den >= 1e-12 * v2;
    const double inv = rsqrt_pos(v2);
    const double lpc = v2 * rcp_fast(den);  // 1 / w
    n[u] = nv * inv;
#if !DGX_LANE_ARW
    g[u] = v * inv;
#endif
    c1[u] = e.alpha * e.O->inv_mass * lpc * sg;
    c0[u] = 0.5 * e.alpha * lpc * (fdot(av, G) * inv) * sg;
#else
    FastEval fe = pre[u].finish(sdf, rl[u], e.radius);
    double sg = 1.0;
    g[u] = fe.g;
    on[u] = pos - u > lim && fe.cls > 0;
    if (pos - u > lim && fe.cls == 0) {  // near the decision boundary: the exact (bit-exact) query decides
      // (inline: an out-of-line call here measured 25% slower, its ABI spills)
      PointEval pe;
      eval_point(sdf, e, ii[u], xk, Rk, true, pe);
      on[u] = !(pe.rho_d < 0.0);
      if (on[u]) {
        g[u] = pe.q.grad;
        sg = pe.fb ? static_cast<double>(pe.q.sign) : 1.0;
      }
    }
    n[u] = fmul(Rk, g[u]);
    // leak_coef (sim.hpp:107-124): s = c1 (n . a) + c0
    const V3 aa = fcross(rel[u], n[u]);
    const V3 Ia = fmul(e.O->Iw, aa);
    const double w = e.O->inv_mass + fdot(aa, Ia);
    on[u] = on[u] && w >= 1e-12;
    const double lpc = rcp_fast(w);
    c1[u] = e.alpha * e.O->inv_mass * lpc * sg;
    c0[u] = 0.5 * e.alpha * lpc * fdot(aa, G) * sg;
  #endif
  }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    if (on[u]) {
      const double s = fma(c1[u], fdot(n[u], a), c0[u]);
      a = fma3(-s, n[u], a);
      const V3 a_rel = n[u] * s;
#if DGX_LANE_ARW
      outer_acc(aR, rel[u], a_rel);  // world frame: the R node's adjoint is aR R (g = R^T n)
#else
      outer_acc(aR, rel[u], g[u] * s);
#endif
      acc.add(ftT, nt, e.sample_link[ii[u]], a_rel, p[u]);
      add_point_grad(e, ii[u], a_rel);
    }
  }
}

template <class Sdf>
__global__ void __launch_bounds__(kLaneAdjThreads, DGX_LANE_MINB) lane_adj_kernel(const __grid_constant__ KHand H, const __grid_constant__ KObj O,
                                                                   const __grid_constant__ Sdf sdf, const __grid_constant__ KSim S,
                                                                   const __grid_constant__ KOpt P, const __grid_constant__ KBuf buf,
                                                                   int mode) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int M = S.M, N = H.N, L = H.L;
  const size_t nt = static_cast<size_t>(buf.B) * M;
  const int lane = static_cast<int>(threadIdx.x);  // one warp per CTA
  const size_t t0 = static_cast<size_t>(blockIdx.x) * kLaneAdjThreads;
  const size_t t = t0 + lane;
  // every lane stays to the end (the warp stages points together); lanes past
  // the batch, of skipped candidates or of sims without an adjoint idle
  const bool in = t < nt;
  const size_t tc = in ? t : nt - 1;
  const int b = static_cast<int>(tc / M), m = static_cast<int>(tc % M);
  const int b_first = static_cast<int>(t0 / M);
  const size_t t_last = t0 + kLaneAdjThreads - 1 < nt ? t0 + kLaneAdjThreads - 1 : nt - 1;
  const int ncw = static_cast<int>(t_last / M) - b_first + 1;
  // a candidate that failed at an earlier iterate of this call stays there
  const bool skip = !in || (mode == kModeOpt && P.k_begin > P.traj_k0 && buf.status[b] != kOk);
  double* ftT = buf.task_ft + tc;  // entry c of this task: ftT[c * nt]
  if (!skip)
    for (int c = 0; c < 6 * L; ++c) ftT[static_cast<size_t>(c) * nt] = 0.0;

  SimEnv e;
  e.lane = 0;
  e.N = N;
  e.gs = S.gs;
  const double* fkb = buf.fk + static_cast<size_t>(b) * (12 * L + 3 * N);
  e.px = fkb + 12 * L;
  e.py = fkb + 12 * L + N;
  e.pz = fkb + 12 * L + 2 * N;
  e.sample_link = H.sample_link;
  e.L = L;
  e.corr = buf.corr + tc * buf.cap_corr;
  e.slots = buf.slots + tc * buf.slot_stride;
  e.fric_order = buf.fric_order + tc * buf.slot_stride;
  e.cap_corr = buf.cap_corr;
  e.slot_cap = buf.slot_stride;
  e.O = &O;
  e.alpha = S.alpha;
  e.mu = S.mu;
  e.dt = S.dt;
  e.radius = S.radius;
  if (mode == kModeOpt) {
    const int k = P.k_begin;
    e.radius = P.iters > 1 ? P.r0 * (1.0 - static_cast<double>(k) / static_cast<double>(P.iters - 1)) : 0.0;
  }
  e.point_grads = buf.point_grads ? buf.point_grads + tc * N * 3 : nullptr;
  e.pts_global = 1;

  const FwdRec* rec = buf.fwd + tc;
  int status = rec->status;
  double residual = rec->residual;
  // canonical_state (rigid.hpp:29-33) with xdot = v_m; predict (sim.hpp:74-83)
  const double* vv = m < kMaxSims ? S.vel[m] : S.vel_dev + 3 * m;
  const V3 v_m{vv[0], vv[1], vv[2]};
  const V3 prev_x = O.com;
  const Q4 prev_q{1.0, 0.0, 0.0, 0.0};
  const V3 prev_thd{0.0, 0.0, 0.0};
  const V3 pred_xdot = v_m + V3{0.0 * e.dt, 0.0 * e.dt, 0.0 * e.dt};
  const V3 pred_x = prev_x + pred_xdot * e.dt;
  const Q4 pred_q = qnormalized(qmul(quat_exp(prev_thd * e.dt), prev_q));
  bool live = false;  // this lane walks the reverse sweep
  V3 aX{0.0, 0.0, 0.0};
  Q4 aQ{0.0, 0.0, 0.0, 0.0};
  const int ncorr = rec->ncorr;
  if (!skip && status == kOk) {
    const V3 x{rec->x[0], rec->x[1], rec->x[2]};
    const Q4 q{rec->q[0], rec->q[1], rec->q[2], rec->q[3]};
    const bool touched = rec->touched != 0;
    const int nfric = rec->nfric;
    // finalize_velocities (sim.hpp:276-287) and the residual (losses.hpp:47-57)
    V3 xdot, thd;
    Q4 qd{0.0, 0.0, 0.0, 0.0};
    const double inv_dt = 1.0 / e.dt;
    if (!touched) {
      xdot = pred_xdot;
      thd = prev_thd;
    } else {
      xdot = (x - prev_x) * inv_dt;
      qd = qmul(q, qconj(prev_q));
      thd = quat_log(qd) * inv_dt;
    }
    const double n1 = norm(xdot), n2 = norm(thd);
    residual = n1 + n2;
    live = touched;  // untouched: constant loss, zero gradient
    if (live) {
      // ---- adjoint: residual -> finalize
      const V3 a_xdot = n1 > 0.0 ? xdot / n1 : V3{0.0, 0.0, 0.0};
      const V3 a_thd = n2 > 0.0 ? thd / n2 : V3{0.0, 0.0, 0.0};
      aQ = qmul_adj_a(quat_log_adj(qd, a_thd * inv_dt), qconj(prev_q));
      aX = a_xdot * inv_dt;
      // ---- friction, reverse (sim.hpp:188-196): the slot's a_lambda / a_n accumulate
      DGX_ASSERT(nfric >= 0 && nfric <= e.slot_cap && ncorr >= 0 && ncorr <= e.cap_corr);
      for (int j = nfric - 1; j >= 0; --j) {
        DGX_ASSERT(e.fric_order[j] >= 0 && e.fric_order[j] < e.slot_cap);
        SlotRec& s = e.slots[e.fric_order[j]];
        double a_lam = s.a_lam;
        V3 a_n{s.a_n[0], s.a_n[1], s.a_n[2]};
        friction_adj(e, prev_x, prev_q, s, aX, aQ, a_lam, a_n);
        s.a_lam = a_lam;
        s.a_n[0] = a_n.x; s.a_n[1] = a_n.y; s.a_n[2] = a_n.z;
      }
    }
  }
  // ---- sweeps, reverse: runs of frozen state between logged corrections.
  // The warp walks positions gs N - 1 .. 0 in lockstep; the points of each
  // block of 32 positions are staged in shared memory for the warp's
  // candidates (cp.async, double-buffered: the next block is in flight while
  // this one is processed).
  if (__any_sync(kFull, live)) {
    double* sb = reinterpret_cast<double*>(smem);
#if DGX_LANE_PTS_EVICT_FIRST
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
    const int rows = ncw * kLaneRow;  // doubles per buffer
    const int top = S.gs * N - 1;
    auto stage = [&](int blk_top, int bi) {  // positions blk_top - kLaneBlk + 1 .. blk_top into buffer bi
      const int itop = blk_top % N;
      for (int x = lane; x < ncw * 3 * kLaneBlk; x += 32) {
        const int c = x / (3 * kLaneBlk), r = x - 3 * kLaneBlk * c, arr = r / kLaneBlk, j = r - arr * kLaneBlk;
        if (blk_top - j < 0) continue;
        int ij = itop - j;
        if (ij < 0) ij += N;
        const double* src = buf.fk + static_cast<size_t>(b_first + c) * (12 * L + 3 * N) + 12 * L +
                            static_cast<size_t>(arr) * N + ij;
        DGX_ASSERT(c < lane_cands_per_warp(M) && ij >= 0 && ij < N && b_first + c < buf.B);
        const double* dst = sb + bi * rows + c * kLaneRow + arr * kLaneRowArr + j;
        const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
#if DGX_LANE_PTS_EVICT_FIRST
        // each sweep streams every candidate's points once (~0.4 GB at config 3):
        // evict-first in L2 so they do not displace the grid cells
        asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(sa), "l"(src), "l"(pol)
                     : "memory");
#else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(src) : "memory");
#endif
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int k = ncorr - 1;
    V3 xk = pred_x;
    Q4 qk = pred_q;
    auto load_state = [&](int kk) {
      xk = pred_x;
      qk = pred_q;
      if (kk >= 0) {
        const CorrRec& c = e.corr[kk];
        xk = V3{c.x[0], c.x[1], c.x[2]};
        qk = Q4{c.q[0], c.q[1], c.q[2], c.q[3]};
      }
    };
    // theta-axpy coefficient G = Iw^T H, H . k == ([0,k] (x) q_k) . aQ
    auto g_of = [&](Q4 qq, Q4 aq) {
      const V3 Hh{-qq.x * aq.w + qq.w * aq.x - qq.z * aq.y + qq.y * aq.z,
                  -qq.y * aq.w + qq.z * aq.x + qq.w * aq.y - qq.x * aq.z,
                  -qq.z * aq.w - qq.y * aq.x + qq.x * aq.y + qq.w * aq.z};
      return ftmul(e.O->Iw, Hh);
    };
    if (live) load_state(k);
    M3 Rk = rotation_matrix(qk);
    V3 G = g_of(qk, aQ);
    int next_f = live && k >= 0 ? e.corr[k].f : -1;
    M3 aR;
    for (int r = 0; r < 9; ++r) aR.m[r] = 0.0;
    LaneFt acc;
    int i = N - 1;
#if DGX_LANE_PTS_FK
    FkPts fkp{H.samples, H.sample_link, fkb};
    (void)sb;
    (void)rows;
#else
    stage(top, 0);
#endif
    int blk = 0, blk_top = top, blk_next = top;
    const double* ps = sb;
    for (int pos = top; pos >= 0; pos -= kLaneU) {
      if (!DGX_LANE_PTS_FK && pos == blk_next) {  // next block: stage the one after it, wait for this one
        blk_next = pos - kLaneBlk;
        __syncwarp();  // every lane is done with the buffer about to be refilled
        if (pos - kLaneBlk >= 0) stage(pos - kLaneBlk, (blk + 1) & 1);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group 1;" ::: "memory");
        __syncwarp();
        ps = sb + (blk & 1) * rows + (b - b_first) * kLaneRow;
        blk_top = pos;
        ++blk;
      }
      if (live) {
#if DGX_LANE_PTS_FK
        lane_leak_steps<kLaneU>(sdf, e, pos, i, max(next_f, pos - kLaneU), xk, Rk, G, aX, aR, acc, ftT, nt, fkp);
#else
        StagedPts sp{ps, blk_top};
        lane_leak_steps<kLaneU>(sdf, e, pos, i, max(next_f, pos - kLaneU), xk, Rk, G, aX, aR, acc, ftT, nt, sp);
#endif
        // this lane's logged corrections inside the window (divergent; rare)
        while (next_f >= 0 && next_f > pos - kLaneU) {  // (next_f = -1: no more corrections)
          const int f = next_f;
          // R node of the state after correction k (read by the run above it)
#if DGX_LANE_ARW
          {
            M3 aRk;  // aR R_k
            for (int r = 0; r < 3; ++r)
              for (int cc = 0; cc < 3; ++cc)
                aRk.m[3 * r + cc] = fma(aR.m[3 * r + 2], Rk.m[6 + cc], fma(aR.m[3 * r + 1], Rk.m[3 + cc], aR.m[3 * r] * Rk.m[cc]));
            aQ = qadd(aQ, rotmat_adj(qk, aRk));
          }
#else
          aQ = qadd(aQ, rotmat_adj(qk, aR));
#endif
          DGX_ASSERT(k >= 0 && k < e.cap_corr && f >= 0 && f <= pos);
          const CorrRec& c = e.corr[k];
          DGX_ASSERT(c.slot >= 0 && c.slot < e.slot_cap);
          const SlotRec& sl = e.slots[c.slot];
          load_state(k - 1);
          bool ok = true;
          const CorrLin o = correction_linear(e, c, xk, qk, aX, aQ, sl.a_lam,
                                              sl.last_corr == k ? V3{sl.a_n[0], sl.a_n[1], sl.a_n[2]}
                                                                : V3{0.0, 0.0, 0.0},
                                              ok);
          if (!ok) status = kReplayMismatch;
          aX = o.aX;
          aQ = o.aQ;
#if DGX_LANE_ARW
          {  // the R node of the state before it, as the world-frame accumulator o.aR R_{k-1}^T
            const M3 Rb = rotation_matrix(qk);
            for (int r = 0; r < 3; ++r)
              for (int cc = 0; cc < 3; ++cc)
                aR.m[3 * r + cc] = fma(o.aR.m[3 * r + 2], Rb.m[3 * cc + 2],
                                       fma(o.aR.m[3 * r + 1], Rb.m[3 * cc + 1], o.aR.m[3 * r] * Rb.m[3 * cc]));
          }
#else
          aR = o.aR;  // R node of the state before it (continued by the run below)
#endif
          {
            const int ip = f % N;
            const V3 pp{e.px[ip], e.py[ip], e.pz[ip]};
            double* d = ftT + static_cast<size_t>(6 * e.sample_link[ip]) * nt;
            const V3 tq = cross(pp, o.a_rel);
            d[0] += o.a_rel.x; d[nt] += o.a_rel.y; d[2 * nt] += o.a_rel.z;
            d[3 * nt] += tq.x; d[4 * nt] += tq.y; d[5 * nt] += tq.z;
            add_point_grad(e, ip, o.a_rel);
          }
          --k;
          Rk = rotation_matrix(qk);
          G = g_of(qk, aQ);
          next_f = k >= 0 ? e.corr[k].f : -1;
          // the window's positions below the correction, with the state before it
          for (int p2 = f - 1; p2 > pos - kLaneU && p2 > next_f; --p2)
#if DGX_LANE_PTS_FK
            lane_leak_steps<1>(sdf, e, p2, p2 % N, next_f, xk, Rk, G, aX, aR, acc, ftT, nt, fkp);
#else
            lane_leak_steps<1>(sdf, e, p2, p2 % N, next_f, xk, Rk, G, aX, aR, acc, ftT, nt, sp);
#endif
        }
      }
      i -= kLaneU;
      if (i < 0) i += N;
    }
#if !DGX_LANE_PTS_FK
    asm volatile("cp.async.wait_all;" ::: "memory");
#endif
    if (live) {
      acc.flush(ftT, nt);
      if (S.discard) {  // this sim's logs are consumed
        l2_discard(e.corr, static_cast<size_t>(ncorr) * sizeof(CorrRec), 0, 1);
        l2_discard(e.slots, static_cast<size_t>(rec->nslot) * sizeof(SlotRec), 0, 1);
      }
    }
  }
  if (skip) return;
  buf.task_res[t] = residual;
  buf.task_stat[t] = status;
  if (buf.sim_res) buf.sim_res[t] = residual;
}

// Per-candidate epilogue after lane_adj_kernel: one warp per candidate.
// Shared memory per warp (doubles): ft_all [M][6L], sres [M], sflag [M] (ints
// in M doubles), scratch [6L + kMaxDim], sg [96], sq [40].
__host__ __device__ inline int lane_epi_doubles(int M, int L) { return M * 6 * L + 2 * M + 6 * L + kMaxDim + 96 + 40; }

__global__ void __launch_bounds__(32 * kEpiWarps) lane_epi_kernel(const __grid_constant__ KHand H, const __grid_constant__ KSim S,
                                                                  const __grid_constant__ KOpt P, const __grid_constant__ KBuf buf, int mode) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int M = S.M, N = H.N, L = H.L, J = H.J, D = 6 + J, Qd = 7 + J;
  const int b = static_cast<int>(blockIdx.x) * static_cast<int>(blockDim.x >> 5) + warp;
  if (b >= buf.B) return;  // warp-uniform
  if (mode == kModeOpt && P.k_begin > P.traj_k0 && buf.status[b] != kOk) return;
  double* wb = reinterpret_cast<double*>(smem) + static_cast<size_t>(warp) * lane_epi_doubles(M, L);
  double* ft_all = wb;
  double* sres = ft_all + M * 6 * L;
  int* sflag = reinterpret_cast<int*>(sres + M);
  double* scratch = sres + 2 * M;
  double* sg = scratch + 6 * L + kMaxDim;
  double* sq = sg + 96;
  const size_t nt = static_cast<size_t>(buf.B) * M, b0 = static_cast<size_t>(b) * M;
  for (int x = lane; x < M * 6 * L; x += 32) {
    const int mm = x / (6 * L), c = x - mm * 6 * L;
    ft_all[x] = __ldcg(buf.task_ft + static_cast<size_t>(c) * nt + b0 + mm);
  }
  for (int x = lane; x < M; x += 32) {
    sres[x] = __ldcg(buf.task_res + b0 + x);
    sflag[x] = __ldcg(buf.task_stat + b0 + x);
  }
  if (lane < Qd) sq[lane] = buf.q[static_cast<size_t>(b) * Qd + lane];
  double am = 0.0, av = 0.0, b1t = 1.0, b2t = 1.0;
  if (mode == kModeOpt) {
    if (lane < D) {
      am = buf.adam_m[static_cast<size_t>(b) * D + lane];
      av = buf.adam_v[static_cast<size_t>(b) * D + lane];
    }
    for (int kk = 0; kk < P.k_begin; ++kk) { b1t = b1t * P.beta1; b2t = b2t * P.beta2; }
  }
  __syncwarp();
  const double* link = buf.fk + static_cast<size_t>(b) * (12 * L + 3 * N);
  if (buf.sim_grads && mode != kModeEval) {  // debug: per-perturbation gradient via the FK adjoint
    for (int mm = 0; mm < M; ++mm) {
      for (int x = lane; x < 6 * L; x += 32) scratch[x] = ft_all[mm * 6 * L + x];
      __syncwarp();
      fk_adjoint(H, sq, link, scratch, sg, lane);
      for (int x = lane; x < D; x += 32) buf.sim_grads[(b0 + mm) * D + x] = sg[x];
      __syncwarp();
    }
  }
  int cand_status = kOk;
  const int k = mode == kModeOpt ? P.k_begin : 0;
  candidate_epilogue(H, S, P, buf, mode, b, k, lane, sflag, sres, ft_all, link, scratch, sg, sq, am, av, b1t, b2t,
                     cand_status);
  __syncwarp();
  if (mode == kModeOpt) {
    if (lane < Qd) buf.q[static_cast<size_t>(b) * Qd + lane] = sq[lane];
    if (lane < D) {
      buf.adam_m[static_cast<size_t>(b) * D + lane] = am;
      buf.adam_v[static_cast<size_t>(b) * D + lane] = av;
    }
  }
  if (lane == 0) buf.status[b] = cand_status;
  __syncwarp();
  if (S.discard) l2_discard(link, sizeof(double) * (12 * L + 3 * N), lane, 32);  // FK record consumed
}
