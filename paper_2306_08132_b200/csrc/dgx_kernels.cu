// dgx_kernels.cu — the fused batched grasp-search kernel for sm_100a.
//
// One CTA per grasp candidate (persistent grid-stride), one warp per
// perturbation simulation (M = 7, losses.hpp:21-27). Per candidate-iteration:
//
//   1. FK (HandModel::forward<Rec>, hand.hpp:116-152; record_pose_vars,
//      hand.cpp:246-257) -> world points in shared memory (SoA, FP64).
//   2. Per warp: predict (sim.hpp:74-83), then the Gauss-Seidel contact solve
//      (ContactSolver::solve, sim.hpp:138-210) with SPECULATIVE lanes: 32
//      consecutive points are evaluated against the current state, the first
//      active lane (ballot) is applied serially, evaluation restarts right after
//      it. Inactive points never change forward values (the zero-depth axpy,
//      sim.hpp:105-125), so this reproduces the sequential sweep exactly.
//      Friction (sim.hpp:247-274) in point order, finalize (sim.hpp:276-287),
//      residual |xdot| + |thetadot| (losses.hpp:47-57).
//   3. Per warp: hand-written adjoint of the recorded path (the reference tape,
//      tape.cpp:27-114): residual -> finalize -> friction (reverse) -> sweeps in
//      reverse. Only active corrections are logged; inactive runs between them
//      are recomputed and their leak channel (sim.hpp:105-125, gate backward
//      -alpha, tape.hpp:179-185) is a 3-vector affine recurrence on adj_x.
//      Point adjoints are folded straight into per-link force/torque sums.
//   4. Warp 0: FK adjoint (per-joint a_j . (T_sub - o_j x F_sub)), qrange /
//      qlimit (losses.hpp:70-93), the losses.cpp:20-66 reductions, and for
//      the optimizer the shared App. C driver (Adam + apply_gradient_step,
//      losses.cpp:92-102).
//
// Built with --fmad=false: every forward value is the same IEEE op sequence
// as the reference, so activations / corrections are bit-exact. Adjoint code
// uses explicit fma().
#include <type_traits>
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>

// 32-position groups the forward classifies per iteration (A/B knob; measured
// forward ms per step, config 3 / config 2 / config 4: 1 group 15.12 / 1.35 /
// 2.46, 2 groups 15.62 / 1.40 / 2.49, 3-4 groups slower)
// out-of-line rare forward paths (A/B knobs)
#ifndef DGX_CORR_INLINE
#define DGX_CORR_INLINE __device__ __forceinline__
#endif
#ifndef DGX_FRIC_INLINE
#define DGX_FRIC_INLINE __device__ __forceinline__
#endif
#ifndef DGX_FWD_HALVES
#define DGX_FWD_HALVES 1
#endif
static constexpr int kFwdHalves = DGX_FWD_HALVES;

// global-points forward: prefetch the next chunk's points into L1 (A/B knob;
// measured slower: config-3 forward 17.5 -> 18.5 ms)
#ifndef DGX_FWD_PREFETCH
#define DGX_FWD_PREFETCH 0
#endif

#ifdef DGX_PROFILE_REGIONS
namespace dgx {
__device__ unsigned long long g_prof[48];
}
// mesh traversal counters (lane 0 of each warp): 23 nearest queries, 24
// nearest node pops, 25 ray casts, 26 ray node pops, 27 exact queries
#define DGX_MESH_CNT(r, n) \
  if ((threadIdx.x & 31) == 0) atomicAdd(&dgx::g_prof[r], static_cast<unsigned long long>(n))
#endif
#include "dgx_adjoint.cuh"
#include "dgx_kernel.cuh"
#include "dgx_sdf_fast.cuh"

namespace dgx {

constexpr unsigned kFull = 0xffffffffu;

// Optional region timers (profiling builds only: -DDGX_PROFILE_REGIONS).
// Lane 0 of each warp accumulates clock64() cycles / event counts per region.
#ifdef DGX_PROFILE_REGIONS
#define PROF_T(v) const long long v = clock64()
#define PROF_ACC(r, v) \
  if ((threadIdx.x & 31) == 0) atomicAdd(&g_prof[r], static_cast<unsigned long long>(clock64() - (v)))
#define PROF_CNT(r, n) \
  if ((threadIdx.x & 31) == 0) atomicAdd(&g_prof[r], static_cast<unsigned long long>(n))
#else
#define PROF_T(v)
#define PROF_ACC(r, v)
#define PROF_CNT(r, n)
#endif

__device__ __forceinline__ double shfl(double v, int l) { return __shfl_sync(kFull, v, l); }
__device__ __forceinline__ V3 shfl(V3 v, int l) { return V3{shfl(v.x, l), shfl(v.y, l), shfl(v.z, l)}; }
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) {
    double w = __shfl_xor_sync(kFull, v, o);
    v = v < w ? w : v;
  }
  return v;
}

// Scratch that has been consumed (correction logs / matrices, contact slots,
// the forward's FK record) is dead until rewritten: drop its L2 lines without
// write-back (PTX discard.global.L2, sm_80+) so it never costs HBM writes nor
// evicts the SDF cells. Only whole 128 B lines inside [p, p + bytes) are
// discarded; callers have finished every read of the range.
__device__ __forceinline__ void l2_discard(const void* p, size_t bytes, int part, int nparts) {
  const uintptr_t a = (reinterpret_cast<uintptr_t>(p) + 127) & ~static_cast<uintptr_t>(127);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes) & ~static_cast<uintptr_t>(127);
  for (uintptr_t l = a + 128 * static_cast<uintptr_t>(part); l < e; l += 128 * static_cast<uintptr_t>(nparts))
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(l) : "memory");
}

struct SimEnv {
  int lane, N, gs, seg_max;
  const double *px, *py, *pz;
  const int* sample_link;
  unsigned* bitmap;
  int* slot_of_point;     // [N] slot index, valid where the bitmap bit is set
  double* stage;
  double* ft;             // [L*6] this warp's link force / torque accumulators (shared)
  double* gft;            // [L*6] this warp's global spill buffer for the adjoint walk
  int L;
  CorrRec* corr;
  SlotRec* slots;
  int* fric_order;
  int cap_corr;
  double* cmat;           // [cap_corr, kCorrMat] batched correction reverse (this warp)
  const KObj* O;          // mass / COM / world inverse inertia (kernel parameter space)
  double radius, alpha, mu, dt;
  double* point_grads;    // debug, may be null
  int* mcache;            // mesh: [gs*N] packed (face, sign) of the forward's query per point-sweep
  double* mcert;          // mesh: [N,4] nearest-face certificates (reset per sim)
  int* mcf;               // mesh: [N, 1 + kCertFaces]
  int fold;               // warp-task adjoint: fold the identical final sweeps
  int discard;            // KSim::discard
  int slot_cap;           // contact-slot / friction-order entries of this sim's logs
  int pts_global;         // px / py / pz point into global memory (global-points forward)
};

// Forward classification of grids through the FP32 pre-filter (see
// grid_inactive_f32); the other backends classify in FP64.
template <class Sdf>
constexpr bool kF32Prefilter = false;
template <>
constexpr bool kF32Prefilter<GridSdf> = true;

// Classification of flattened position fpos (sweep*N + i) at r (FMA-built
// r_local). Mesh objects: the forward's exact query is warm-started from the
// point's face one sweep earlier and its (face, sign) recorded; the adjoint
// re-evaluates that face only. Both see the same state and r, so they
// reproduce the forward's decision and gradient exactly.
template <class Sdf>
__device__ __forceinline__ FastEval classify_fwd(const Sdf& sdf, const SimEnv& e, int, V3 r) {
  return classify(sdf, r, e.radius);
}
template <class Sdf>
__device__ __forceinline__ FastEval classify_bwd(const Sdf& sdf, const SimEnv& e, int, V3 r) {
  return classify(sdf, r, e.radius);
}
__device__ __forceinline__ FastEval classify_fwd(const MeshSdf& m, const SimEnv& e, int fpos, V3 r) {
  const int hint = fpos >= e.N ? (e.mcache[fpos - e.N] >> 1) : -1;
  const int i = fpos % e.N;
  int packed;
  const SdfQuery q = m.query_cert(r, hint, packed, e.mcert + 4 * i, e.mcf + (kCertFaces + 1) * i);
  e.mcache[fpos] = packed;
  return classify_query(q, r, e.radius);
}
__device__ __forceinline__ FastEval classify_bwd(const MeshSdf& m, const SimEnv& e, int fpos, V3 r) {
  return classify_query(m.query_packed(r, e.mcache[fpos]), r, e.radius);
}

struct PointEval {
  V3 p, rel, rl;
  SdfQuery q;
  double rho_d;
  bool fb;
};

// rel = p - x; r_local = R^T rel + com (sim.hpp:160-161); dilated SDF value in
// recorded (sdf.cpp:83-107) or forward-only (sdf.cpp:69-81) semantics.
template <class Sdf>
__device__ __forceinline__ void eval_point(const Sdf& sdf, const SimEnv& e, int i, V3 x, const M3& R,
                                           bool record, PointEval& pe) {
  DGX_ASSERT(i >= 0 && i < e.N);
  pe.p = V3{e.px[i], e.py[i], e.pz[i]};
  pe.rel = pe.p - x;
  pe.rl = tmul(R, pe.rel) + e.O->com;
  if (!record && sdf_culled(sdf, pe.rl, e.radius)) {  // dilated_within -> nullopt: inactive (sim.hpp:177-178)
    pe.q = SdfQuery{kInf, V3{0.0, 0.0, 1.0}, pe.rl, 1};
    pe.fb = false;
    pe.rho_d = kInf;
    return;
  }
  pe.q = sdf.query(pe.rl);
  pe.fb = fabs(pe.q.rho) < kSurfaceEps;
  if (record && pe.fb) {
    V3 dx = pe.rl - pe.q.proxy;
    double proj = dx.x * pe.q.grad.x + dx.y * pe.q.grad.y + dx.z * pe.q.grad.z;
    pe.rho_d = static_cast<double>(pe.q.sign) * proj - e.radius;
  } else {
    pe.rho_d = pe.q.rho - e.radius;
  }
}

// Per-lane accumulator of d/dp folded into per-link force / torque sums
// (F_l = sum adj_p, T_l = sum p x adj_p). When a lane's walk moves to another
// link it spills its partial to the warp's global link buffer with native
// FP64 reductions (RED.ADD.F64: fire-and-forget, no shared-memory CAS); the
// buffer is folded into the shared sums once per perturbation sim.
struct FtAcc {
  int link = -1;
  V3 F{0.0, 0.0, 0.0}, T{0.0, 0.0, 0.0};
  __device__ __forceinline__ void reset() {
    link = -1;
    F = V3{0.0, 0.0, 0.0};
    T = V3{0.0, 0.0, 0.0};
  }
  __device__ __forceinline__ void spill(double* ft) {
    DGX_ASSERT(link >= 0 && link < 32);
    double* d = ft + 6 * link;
    atomicAdd(d + 0, F.x); atomicAdd(d + 1, F.y); atomicAdd(d + 2, F.z);
    atomicAdd(d + 3, T.x); atomicAdd(d + 4, T.y); atomicAdd(d + 5, T.z);
    reset();
  }
  __device__ __forceinline__ void spill_if_any(double* ft) {
    if (link >= 0) spill(ft);
  }
  __device__ __forceinline__ void add(double* ft, int l, V3 ap, V3 p) {
    if (l != link) {
      if (link >= 0) spill(ft);
      link = l;
    }
    F = F + ap;
    T = T + fcross(p, ap);
  }
};

// Warp-cooperative flush of the per-lane link accumulators. Lanes walk
// positions in descending order, so equal links normally occupy one
// contiguous lane range: a single segmented inclusive scan then leaves each
// segment's sum in its highest lane, which writes it (one writer per link, no
// atomics). Non-contiguous key patterns (possible only for tiny hands) take
// the keyed butterfly loop instead.
__device__ __forceinline__ void ft_flush_warp(FtAcc& acc, double* ft, int lane) {
  const int key = acc.link;
  const unsigned m = __match_any_sync(0xffffffffu, key);
  const int lo = __ffs(m) - 1;
  const unsigned run = m >> lo;
  if (__all_sync(0xffffffffu, (run & (run + 1u)) == 0u)) {
    double v[6] = {acc.F.x, acc.F.y, acc.F.z, acc.T.x, acc.T.y, acc.T.z};
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      double u[6];
#pragma unroll
      for (int k = 0; k < 6; ++k) u[k] = __shfl_up_sync(0xffffffffu, v[k], d);
      if (lane - d >= lo) {
#pragma unroll
        for (int k = 0; k < 6; ++k) v[k] += u[k];
      }
    }
    if (key >= 0 && lane == 31 - __clz(m)) {
      double* d = ft + 6 * key;
#pragma unroll
      for (int k = 0; k < 6; ++k) d[k] += v[k];
    }
  } else {
    unsigned pending = __ballot_sync(0xffffffffu, key >= 0);
    while (pending) {
      const int leader = __ffs(pending) - 1;
      const int kk = __shfl_sync(0xffffffffu, key, leader);
      const bool mine = key == kk;
      pending &= ~__ballot_sync(0xffffffffu, mine);
      double v[6] = {mine ? acc.F.x : 0.0, mine ? acc.F.y : 0.0, mine ? acc.F.z : 0.0,
                     mine ? acc.T.x : 0.0, mine ? acc.T.y : 0.0, mine ? acc.T.z : 0.0};
#pragma unroll
      for (int k = 0; k < 6; ++k)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
      if (lane == leader) {
        double* d = ft + 6 * kk;
#pragma unroll
        for (int k = 0; k < 6; ++k) d[k] += v[k];
      }
    }
  }
  __syncwarp();
  acc.reset();
}

__device__ __forceinline__ void add_point_grad(const SimEnv& e, int i, V3 ap) {
  if (e.point_grads) {
    atomicAdd(e.point_grads + 3 * i, ap.x);
    atomicAdd(e.point_grads + 3 * i + 1, ap.y);
    atomicAdd(e.point_grads + 3 * i + 2, ap.z);
  }
}

struct SimStats {
  int active = 0, corrections = 0, singular = 0;
  double max_pen = 0.0, max_fric = 0.0;
};

// ContactSolver::apply_friction (sim.hpp:247-274) on values; returns whether
// the state changed. Friction-ratio stat as sim.hpp:266-272.
DGX_FRIC_INLINE bool friction_fwd(const SimEnv& e, V3 prev_x, Q4 prev_q, V3& x, Q4& q, V3 rb, V3 n,
                                             double lambda_n, SimStats& st, Q4& E, double& sin_half) {
  V3 before = prev_x + rotate(prev_q, rb);
  V3 arm = rotate(q, rb);
  V3 after = x + arm;
  V3 u = after - before;
  V3 u_t = u - n * dot(u, n);
  double ut = norm(u_t);
  if (ut < 1e-12) return false;
  V3 t = u_t / ut;
  V3 at = cross(arm, t);
  V3 iwat = mul(e.O->Iw, at);
  double w_t = e.O->inv_mass + dot(at, iwat);
  if (w_t < 1e-12) return false;
  double a1 = ut / w_t, a2 = e.mu * lambda_n;
  double lam_t = a1 <= a2 ? a1 : a2;
  x = x - t * (e.O->inv_mass * lam_t);
  E = quat_exp_sin(iwat * (-lam_t), sin_half);
  q = qnormalized(qmul(E, q));
  ++st.corrections;
  double denom = e.mu * lambda_n;
  if (denom > 0.0) {
    double r = lam_t / denom;
    st.max_fric = st.max_fric < r ? r : st.max_fric;
  }
  return true;
}

// Reverse of friction_fwd for one applied slot; aX/aQ: adjoints of the state
// after it (in) and before it (out). Accumulates the slot's a_lam / a_n.
__device__ __forceinline__ void friction_adj(const SimEnv& e, V3 prev_x, Q4 prev_q, const SlotRec& s, V3& aX, Q4& aQ,
                                             double& a_lam_slot, V3& a_n_slot, V3* a_prev_x = nullptr,
                                             Q4* a_prev_q = nullptr) {
  V3 rb{s.rb[0], s.rb[1], s.rb[2]};
  V3 n{s.n[0], s.n[1], s.n[2]};
  V3 fx{s.fx[0], s.fx[1], s.fx[2]};
  Q4 fq{s.fq[0], s.fq[1], s.fq[2], s.fq[3]};
  V3 before = prev_x + rotate(prev_q, rb);
  V3 arm = rotate(fq, rb);
  V3 u = (fx + arm) - before;
  double d = dot(u, n);
  V3 u_t = u - n * d;
  double ut = norm(u_t);
  V3 t = u_t / ut;
  V3 at = cross(arm, t);
  V3 iwat = mul(e.O->Iw, at);
  double w_t = e.O->inv_mass + dot(at, iwat);
  double a1 = ut / w_t, a2 = e.mu * s.lambda_n;
  bool first = a1 <= a2;
  double lam_t = first ? a1 : a2;
  V3 om = iwat * (-lam_t);
  const Q4 E{s.fE[0], s.fE[1], s.fE[2], s.fE[3]};  // logged by the forward
  Q4 P = qmul(E, fq);
  // x_out = fx - t (m^-1 lam_t)
  V3 a_t = aX * (-e.O->inv_mass * lam_t);
  double a_lamt = -e.O->inv_mass * fdot(t, aX);
  // q_out = normalized(E (x) fq)
  Q4 a_P = qnormalize_adj(P, aQ);
  Q4 a_E = qmul_adj_a(a_P, fq);
  Q4 aQ_in = qmul_adj_b(a_P, E);
  V3 a_om = quat_exp_adj_sc(om, a_E, s.fsin, E.w);
  a_lamt -= fdot(iwat, a_om);
  V3 a_iwat = a_om * (-lam_t);
  double a_a1 = first ? a_lamt : 0.0;
  double a_a2 = first ? 0.0 : a_lamt;
  a_lam_slot = fma(e.mu, a_a2, a_lam_slot);
  double a_ut = a_a1 / w_t;
  double a_wt = -a_a1 * a1 / w_t;
  V3 a_at = iwat * a_wt;
  a_iwat = fma3(a_wt, at, a_iwat);
  a_at = a_at + ftmul(e.O->Iw, a_iwat);
  V3 a_arm = cross(t, a_at);
  a_t = a_t + cross(a_at, arm);
  V3 a_utv = a_t / ut;
  a_ut -= fdot(a_t, t) / ut;
  a_utv = fma3(a_ut / ut, u_t, a_utv);
  V3 a_u = a_utv;
  V3 a_n = a_utv * (-d);
  double a_d = -fdot(n, a_utv);
  a_u = fma3(a_d, n, a_u);
  a_n = fma3(a_d, u, a_n);
  a_n_slot = a_n_slot + a_n;
  aX = aX + a_u;
  a_arm = a_arm + a_u;
  Q4 r = rotate_adj_q(fq, rb, a_arm);
  aQ = qadd(aQ_in, r);
  if (a_prev_x) {  // before = prev.x + rotate(prev.theta, r_body) (sim.hpp:250): a_before = -a_u
    const V3 ab = a_u * -1.0;
    *a_prev_x = *a_prev_x + ab;
    *a_prev_q = qadd(*a_prev_q, rotate_adj_q(prev_q, rb, ab));
  }
}

// Warp-wide all-reduce of a per-lane 3x3 accumulator.
__device__ __forceinline__ M3 warp_sum(const M3& A) {
  M3 r;
  for (int k = 0; k < 9; ++k) r.m[k] = warp_sum(A.m[k]);
  return r;
}

// 1/w to full double accuracy: MUFU reciprocal seed + two Newton steps
// (adjoint-only; the forward keeps IEEE division)
__device__ __forceinline__ double rcp_fast(double w) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(w));
  double e = fma(-w, r, 1.0);
  r = fma(r, e, r);
  e = fma(-w, r, 1.0);
  return fma(r, e, r);
}

// Geometry of one inactive point-sweep for the leak adjoint (sim.hpp:105-125
// recorded with C = gate(rho_d) = 0): unit SDF gradient g (local frame),
// n = R g (world), the arm rel = p - x. contrib == false for points that were
// active in the forward (a singular-skipped correction: no axpy recorded).
struct LeakGeo {
  V3 p, rel, g, n;
  double sg;     // sign factor of the interpolated-normal fallback (sdf.cpp:92-98)
  bool contrib;
};

template <class Sdf>
__device__ __forceinline__ void leak_geo(const Sdf& sdf, const SimEnv& e, int i, int fpos, V3 xk, const M3& Rk,
                                         LeakGeo& L) {
  DGX_ASSERT(i >= 0 && i < e.N);
  L.p = V3{e.px[i], e.py[i], e.pz[i]};
  L.rel = L.p - xk;
  const V3 rl = ftmul_add(Rk, L.rel, e.O->com);
  FastEval fe = classify_bwd(sdf, e, fpos, rl);
  L.sg = 1.0;
  L.contrib = false;
  if (fe.cls == 0) {  // near the decision boundary: the exact (bit-exact) query decides
    PointEval pe;
    eval_point(sdf, e, i, xk, Rk, true, pe);
    if (pe.rho_d < 0.0) return;
    fe.g = pe.q.grad;
    L.sg = pe.fb ? static_cast<double>(pe.q.sign) : 1.0;
  } else if (fe.cls < 0) {
    return;
  }
  L.g = fe.g;
  L.n = fmul(Rk, fe.g);
  L.contrib = true;
}

// Leak recurrence coefficients: adj_x_before = adj_x_after - s n with
// s = c1 (n . adj_x_after) + c0 (kx = -(m^-1/w) n, g_q = 1/2 [0,k_w] (x) q,
// gate backward -alpha; sim.hpp:107-124, tape.cpp:103-107).
__device__ __forceinline__ bool leak_coef(const SimEnv& e, const LeakGeo& L, V3 G, double& c1, double& c0) {
  const V3 a = fcross(L.rel, L.n);
  const V3 Ia = fmul(e.O->Iw, a);
  const double w = e.O->inv_mass + fdot(a, Ia);
  if (w < 1e-12) return false;
  const double lpc = rcp_fast(w);
  c1 = e.alpha * e.O->inv_mass * lpc * L.sg;
  c0 = 0.5 * e.alpha * lpc * fdot(a, G) * L.sg;
  return true;
}

// per (segment slot, lane): c1, c0, g.x, g.y, g.z staged in shared memory by pass 1
__device__ __forceinline__ int stg_idx(int k, int c, int lane) { return (k * 5 + c) * 32 + lane; }

// Adjoint of one inactive run [lo, hi) of flattened (sweep*N + point)
// positions with frozen state (xk, qk): lane l walks positions
// [top-(l+1)S, top-lS) downward. Pass 1 composes each lane's affine map on
// adj_x, a 5-level Kogge-Stone scan hands every lane its incoming adj_x,
// pass 3 re-walks with it and emits the point / R adjoints.
template <class Sdf>
__device__ void process_run(const Sdf& sdf, SimEnv& e, int lo, int hi, V3 xk, Q4 qk, const M3& Rk, Q4 aQ, V3& aX,
                            M3& aR, FtAcc& acc, double c0scale = 1.0, M3* map_out = nullptr,
                            V3* off_out = nullptr) {
  // map_out != nullptr: map-only mode. No contributions are emitted; the
  // run's composed affine map on adj_x (a -> M a + b) is returned instead.
  // c0scale multiplies the constant (theta-channel) term of every point, so a
  // run fed with sum_k X_k and c0scale = K emits the sum over K identical runs.
  const int lane = e.lane, N = e.N;
  double* stg = e.stage;
  PROF_CNT(35, map_out ? 0 : hi - lo);
  // H . k == ([0,k] (x) q_k) . aQ ; G = Iw^T H  (theta-axpy coefficient)
  const V3 H{-qk.x * aQ.w + qk.w * aQ.x - qk.z * aQ.y + qk.y * aQ.z,
             -qk.y * aQ.w + qk.z * aQ.x + qk.w * aQ.y - qk.x * aQ.z,
             -qk.z * aQ.w - qk.y * aQ.x + qk.x * aQ.y + qk.w * aQ.z};
  const V3 G = ftmul(e.O->Iw, H);
  V3 X = aX;
  M3 Mtot;
  V3 btot{0.0, 0.0, 0.0};
  for (int t = 0; t < 9; ++t) Mtot.m[t] = (t % 4 == 0) ? 1.0 : 0.0;
  for (int top = hi; top > lo;) {
    // segment length adapts to the run: short runs keep all lanes busy, long
    // runs amortise the scan over up to seg_max points per lane
    const int S = min(e.seg_max, (top - lo + 31) / 32);
    DGX_ASSERT(S >= 1 && S <= e.seg_max && lo >= 0 && top <= e.gs * N);
    const int shi = top - lane * S;
    const int slo = max(top - (lane + 1) * S, lo);
    const int cnt = shi - slo;
    PROF_CNT(18, 1);
    PROF_T(t1a);
#ifdef DGX_P1A_PAIR
    // ---- pass 1a: per point n = R g, c1, c0 -> shared staging (own lane).
    // Two points per step: both classifications are straight-line code so the
    // compiler overlaps their grid loads and FP64 chains; the exact query for
    // undecided points follows (rare).
    int i = cnt > 0 ? (shi - 1) % N : 0;
    for (int k = 0; k < cnt; k += 2) {
      const int i0 = i;
      const int i1 = i0 > 0 ? i0 - 1 : N - 1;
      LeakGeo L[2];
      FastEval fe[2];
      const int ii[2] = {i0, i1};
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        L[u].p = V3{e.px[ii[u]], e.py[ii[u]], e.pz[ii[u]]};
        L[u].rel = L[u].p - xk;
        fe[u] = classify(sdf, ftmul(Rk, L[u].rel) + e.O->com, e.radius);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        L[u].sg = 1.0;
        L[u].contrib = fe[u].cls > 0;
        if (fe[u].cls == 0 && (u == 0 || k + 1 < cnt)) {  // decision boundary: exact (bit-exact) query
          PointEval pe;
          eval_point(sdf, e, ii[u], xk, Rk, true, pe);
          if (!(pe.rho_d < 0.0)) {
            fe[u].g = pe.q.grad;
            L[u].sg = pe.fb ? static_cast<double>(pe.q.sign) : 1.0;
            L[u].contrib = true;
          }
        }
        L[u].g = fe[u].g;
        L[u].n = fmul(Rk, fe[u].g);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (u == 1 && k + 1 >= cnt) break;
        double c1 = 0.0, c0 = 0.0;
        if (!(L[u].contrib && leak_coef(e, L[u], G, c1, c0))) {
          c1 = 0.0;
          c0 = 0.0;
        }
        stg[stg_idx(k + u, 0, lane)] = c1;
        stg[stg_idx(k + u, 1, lane)] = c0;
        stg[stg_idx(k + u, 2, lane)] = L[u].n.x;
        stg[stg_idx(k + u, 3, lane)] = L[u].n.y;
        stg[stg_idx(k + u, 4, lane)] = L[u].n.z;
      }
      i = i1 > 0 ? i1 - 1 : N - 1;
    }
#else
    // ---- pass 1a: per point n = R g, c1, c0 -> shared staging (own lane)
    int i = cnt > 0 ? (shi - 1) % N : 0;
    for (int k = 0; k < cnt; ++k) {
      LeakGeo L;
      leak_geo(sdf, e, i, shi - 1 - k, xk, Rk, L);
      double c1 = 0.0, c0 = 0.0;
      if (!(L.contrib && leak_coef(e, L, G, c1, c0))) {
        c1 = 0.0;
        c0 = 0.0;
      }
      c0 *= c0scale;
      stg[stg_idx(k, 0, lane)] = c1;
      stg[stg_idx(k, 1, lane)] = c0;
      stg[stg_idx(k, 2, lane)] = L.n.x;
      stg[stg_idx(k, 3, lane)] = L.n.y;
      stg[stg_idx(k, 4, lane)] = L.n.z;
      if (--i < 0) i = N - 1;
    }
#endif
    PROF_ACC(6, t1a);
    PROF_T(t1b);
    // ---- pass 1b: this lane's composed map a -> M a + b
    M3 Mm;
    Mm.m[0] = 1.0; Mm.m[1] = 0.0; Mm.m[2] = 0.0;
    Mm.m[3] = 0.0; Mm.m[4] = 1.0; Mm.m[5] = 0.0;
    Mm.m[6] = 0.0; Mm.m[7] = 0.0; Mm.m[8] = 1.0;
    V3 bm{0.0, 0.0, 0.0};
    for (int k = 0; k < cnt; ++k) {
      const double c1 = stg[stg_idx(k, 0, lane)], c0 = stg[stg_idx(k, 1, lane)];
      if (c1 != 0.0 || c0 != 0.0) {
        const V3 n{stg[stg_idx(k, 2, lane)], stg[stg_idx(k, 3, lane)], stg[stg_idx(k, 4, lane)]};
        const V3 v{fma(n.z, Mm.m[6], fma(n.y, Mm.m[3], n.x * Mm.m[0])),
                   fma(n.z, Mm.m[7], fma(n.y, Mm.m[4], n.x * Mm.m[1])),
                   fma(n.z, Mm.m[8], fma(n.y, Mm.m[5], n.x * Mm.m[2]))};
        outer_acc(Mm, n * (-c1), v);
        const double t = fdot(n, bm);
        bm = fma3(-fma(c1, t, c0), n, bm);
      }
    }
    PROF_ACC(7, t1b);
    PROF_T(t2);
    // ---- pass 2: inclusive scan of maps across lanes (lane 0 applies first)
    M3 Mi = Mm;
    V3 bi = bm;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      M3 Mu;
#pragma unroll
      for (int t = 0; t < 9; ++t) Mu.m[t] = __shfl_up_sync(kFull, Mi.m[t], d);
      const V3 bu{__shfl_up_sync(kFull, bi.x, d), __shfl_up_sync(kFull, bi.y, d), __shfl_up_sync(kFull, bi.z, d)};
      if (lane >= d) {
        bi = fmul(Mi, bu) + bi;
        M3 P;
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
          for (int c = 0; c < 3; ++c)
            P.m[3 * r + c] = fma(Mi.m[3 * r + 2], Mu.m[6 + c], fma(Mi.m[3 * r + 1], Mu.m[3 + c], Mi.m[3 * r] * Mu.m[c]));
        Mi = P;
      }
    }
    M3 Mp;
#pragma unroll
    for (int t = 0; t < 9; ++t) Mp.m[t] = __shfl_up_sync(kFull, Mi.m[t], 1);
    const V3 bp{__shfl_up_sync(kFull, bi.x, 1), __shfl_up_sync(kFull, bi.y, 1), __shfl_up_sync(kFull, bi.z, 1)};
    V3 a = lane == 0 ? X : fmul(Mp, X) + bp;
    M3 Ml;
#pragma unroll
    for (int t = 0; t < 9; ++t) Ml.m[t] = __shfl_sync(kFull, Mi.m[t], 31);
    const V3 bl{__shfl_sync(kFull, bi.x, 31), __shfl_sync(kFull, bi.y, 31), __shfl_sync(kFull, bi.z, 31)};
    const V3 Xnext = fmul(Ml, X) + bl;
    __syncwarp();
    PROF_ACC(8, t2);
    if (map_out) {  // map-only: compose this block's map after the previous ones
      btot = fmul(Ml, btot) + bl;
      M3 P;
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
          P.m[3 * r + c] = fma(Ml.m[3 * r + 2], Mtot.m[6 + c], fma(Ml.m[3 * r + 1], Mtot.m[3 + c], Ml.m[3 * r] * Mtot.m[c]));
      Mtot = P;
      X = Xnext;
      top -= 32 * S;
      __syncwarp();
      continue;
    }
    PROF_T(t3);
    // ---- pass 3: re-walk with the incoming adjoint, emit contributions
    i = cnt > 0 ? (shi - 1) % N : 0;
    for (int k = 0; k < cnt; ++k) {
      const double c1 = stg[stg_idx(k, 0, lane)], c0 = stg[stg_idx(k, 1, lane)];
      if (c1 != 0.0 || c0 != 0.0) {
        const V3 n{stg[stg_idx(k, 2, lane)], stg[stg_idx(k, 3, lane)], stg[stg_idx(k, 4, lane)]};
        const V3 g = ftmul(Rk, n);  // R orthonormal: R^T (R g) = g to rounding
        const V3 p{e.px[i], e.py[i], e.pz[i]};
        const V3 rel = p - xk;
        const double s = fma(c1, fdot(n, a), c0);
        a = fma3(-s, n, a);
        const V3 a_rel = n * s;
        outer_acc(aR, rel, g * s);
        acc.add(e.gft, e.sample_link[i], a_rel, p);
        add_point_grad(e, i, a_rel);
      }
      if (--i < 0) i = N - 1;
    }
    X = Xnext;
    top -= 32 * S;
    __syncwarp();
    PROF_ACC(9, t3);
  }
  aX = X;
  if (map_out) {
    *map_out = Mtot;
    *off_out = btot;
  }
}

struct CorrIn {
  V3 x;
  Q4 q;
  V3 rel, g, p, dx;
  double C;
  int ij, f, ncorr, nslot, sign, fb;
};
struct CorrOut {
  V3 x;
  Q4 q;
  int applied, nslot, status, new_contact;
};

// ContactSolver::apply_contact (sim.hpp:215-245) on values for the first
// active point of the window; logs the correction (state after it) and the
// contact slot. Called by all lanes of the warp (identical values); lane 0
// writes the logs.
DGX_CORR_INLINE CorrOut apply_correction(const SimEnv& e, const CorrIn in) {
  CorrOut out;
  out.x = in.x;
  out.q = in.q;
  out.applied = 0;
  out.nslot = in.nslot;
  out.status = kOk;
  out.new_contact = 0;
  const M3 R = rotation_matrix(in.q);
  const V3 n_w = mul(R, in.g);
  const V3 a = cross(in.rel, n_w);
  const V3 iwa = mul(e.O->Iw, a);
  const double w = e.O->inv_mass + dot(a, iwa);
  if (w < 1e-12) return out;  // singular effective mass: skipped, no state change
  const double lam = in.C / w;
  const V3 x = in.x - n_w * (e.O->inv_mass * lam);
  double sin_half;
  const Q4 E = quat_exp_sin(iwa * (-lam), sin_half);
  const Q4 q = qnormalized(qmul(E, in.q));
  const int ij = in.ij;
  const unsigned bit = 1u << (ij & 31);
  const bool was = (e.bitmap[ij >> 5] & bit) != 0u;
  int slot;
  double lambda_n;
  DGX_ASSERT(ij >= 0 && ij < e.N);
  if (!was) {
    slot = in.nslot;  // slots are sized N (sim.hpp:155): never overflows
    DGX_ASSERT(slot < e.slot_cap);
    out.nslot = in.nslot + 1;
    lambda_n = 0.0 + lam;
    if (e.lane == 0) {
      e.bitmap[ij >> 5] |= bit;
      e.slot_of_point[ij] = slot;
      SlotRec& s = e.slots[slot];
      const V3 rb = tmul(rotation_matrix(q), in.p - x);
      s.rb[0] = rb.x; s.rb[1] = rb.y; s.rb[2] = rb.z;
      s.a_lam = 0.0;
      s.a_n[0] = s.a_n[1] = s.a_n[2] = 0.0;
      s.point = ij;
      s.fric = 0;
    }
  } else {
    slot = e.slot_of_point[ij];
    lambda_n = e.slots[slot].lambda_n + lam;
  }
  if (in.ncorr >= e.cap_corr) { out.status = kCorrOverflow; return out; }
  DGX_ASSERT(slot >= 0 && slot < e.slot_cap && in.ncorr >= 0);
  if (e.lane == 0) {
    SlotRec& s = e.slots[slot];
    s.lambda_n = lambda_n;
    s.n[0] = n_w.x; s.n[1] = n_w.y; s.n[2] = n_w.z;
    s.last_corr = in.ncorr;
    CorrRec& c = e.corr[in.ncorr];
    c.x[0] = x.x; c.x[1] = x.y; c.x[2] = x.z;
    c.q[0] = q.w; c.q[1] = q.x; c.q[2] = q.y; c.q[3] = q.z;
    c.lam = lam;
    c.f = in.f;
    c.slot = slot;
    c.g[0] = in.g.x; c.g[1] = in.g.y; c.g[2] = in.g.z;
    c.rel[0] = in.rel.x; c.rel[1] = in.rel.y; c.rel[2] = in.rel.z;
    c.dx[0] = in.dx.x; c.dx[1] = in.dx.y; c.dx[2] = in.dx.z;
    c.rho_d = -in.C;
    c.E[0] = E.w; c.E[1] = E.x; c.E[2] = E.y; c.E[3] = E.z;
    c.sin_half = sin_half;
    c.sign = in.sign;
    c.fb = in.fb;
  }
  __syncwarp();
  out.x = x;
  out.q = q;
  out.applied = 1;
  out.new_contact = lambda_n == lam ? 1 : 0;  // sim.hpp:242
  return out;
}

// Reverse of apply_contact (sim.hpp:215-245) for logged correction k from the
// logged forward values (no SDF query / trig). For fixed forward values it
// maps v = (aX, aQ) after the correction and the slot's (a_lam, a_n) linearly
// to (aX, aQ) before it, the R-node adjoint aR and the point adjoint a_rel;
// `lam_ok` is the replay check of lambda.
struct CorrLin {
  V3 aX;
  Q4 aQ;
  M3 aR;
  V3 a_rel;
};
__device__ __forceinline__ CorrLin correction_linear(const SimEnv& e, const CorrRec& c, V3 xb, Q4 qb, V3 aX, Q4 aQ,
                                                     double a_lam, V3 a_nw, bool& lam_ok) {
  CorrLin o;
  for (int t = 0; t < 9; ++t) o.aR.m[t] = 0.0;
  const M3 Rb = rotation_matrix(qb);
  const V3 g{c.g[0], c.g[1], c.g[2]};
  const V3 rel{c.rel[0], c.rel[1], c.rel[2]};
  const double C = -c.rho_d;
  const V3 n_w = mul(Rb, g);
  const V3 a = cross(rel, n_w);
  const V3 iwa = mul(e.O->Iw, a);
  const double w = e.O->inv_mass + dot(a, iwa);
  const double lam = C / w;
  lam_ok = lam == c.lam;
  const V3 om = iwa * (-lam);
  const Q4 E{c.E[0], c.E[1], c.E[2], c.E[3]};
  const Q4 P = qmul(E, qb);
  const Q4 a_P = qnormalize_adj(P, aQ);
  const Q4 a_E = qmul_adj_a(a_P, qb);
  const Q4 aQb = qmul_adj_b(a_P, E);
  const V3 a_om = quat_exp_adj_sc(om, a_E, c.sin_half, E.w);
  a_lam -= fdot(iwa, a_om);
  V3 a_iwa = a_om * (-lam);
  a_lam -= e.O->inv_mass * fdot(n_w, aX);
  a_nw = fma3(-e.O->inv_mass * lam, aX, a_nw);
  const double a_C = a_lam / w;
  const double a_w = -a_lam * lam / w;
  V3 a_a = iwa * a_w;
  a_iwa = fma3(a_w, a, a_iwa);
  a_a = a_a + ftmul(e.O->Iw, a_iwa);
  V3 a_rel = cross(n_w, a_a);
  a_nw = a_nw + cross(a_a, rel);
  const V3 a_g = ftmul(Rb, a_nw);
  outer_acc(o.aR, a_nw, g);
  const double a_rho = -a_C;  // gate active: dC/drho = -1
  V3 a_rl;
  if (c.fb) {
    a_rl = g * (static_cast<double>(c.sign) * a_rho);
  } else {
    const V3 dx{c.dx[0], c.dx[1], c.dx[2]};
    const double dist = norm(dx);
    const double inv = static_cast<double>(c.sign) / dist;
    double a_dist = static_cast<double>(c.sign) * a_rho;
    a_dist -= fdot(a_g, dx) * inv / dist;
    a_rl = fma3(a_dist / dist, dx, a_g * inv);
  }
  a_rel = a_rel + fmul(Rb, a_rl);
  outer_acc(o.aR, rel, a_rl);
  o.a_rel = a_rel;
  o.aX = aX - a_rel;
  o.aQ = aQb;
  return o;
}

// Batched correction reverse: matrix of correction k, rows (aX 3, aQ 4,
// aR 9, a_rel 3) x columns (aX 3, aQ 4, 1), plus the replay flag.
constexpr int kCorrRows = 19, kCorrCols = 8, kCorrMat = kCorrRows * kCorrCols + 1;
static_assert(kCorrMat == kCorrMatDoubles, "host scratch sizing");

// All corrections' matrices, (correction, column) tasks spread over the warp.
// Column 7 is the constant part: v = 0 with the slot's final a_lam / a_n
// (set by the friction reverse; correction adjoints only read them).
// Corrections [k_lo, k_hi] go to ring entries k % kCorrBatch.
__device__ __forceinline__ void correction_matrices(const SimEnv& e, int k_lo, int k_hi, V3 pred_x, Q4 pred_q) {
#pragma unroll 1
  for (int t = e.lane; t < (k_hi - k_lo + 1) * kCorrCols; t += 32) {
    const int k = k_lo + t / kCorrCols, cb = t % kCorrCols;
    DGX_ASSERT(k < e.cap_corr);
    const CorrRec c = e.corr[k];
    DGX_ASSERT(c.slot >= 0 && c.slot < e.slot_cap);
    V3 xb = pred_x;
    Q4 qb = pred_q;
    if (k >= 1) {
      const CorrRec& cp = e.corr[k - 1];
      xb = V3{cp.x[0], cp.x[1], cp.x[2]};
      qb = Q4{cp.q[0], cp.q[1], cp.q[2], cp.q[3]};
    }
    V3 vx{cb == 0 ? 1.0 : 0.0, cb == 1 ? 1.0 : 0.0, cb == 2 ? 1.0 : 0.0};
    Q4 vq{cb == 3 ? 1.0 : 0.0, cb == 4 ? 1.0 : 0.0, cb == 5 ? 1.0 : 0.0, cb == 6 ? 1.0 : 0.0};
    double a_lam = 0.0;
    V3 a_nw{0.0, 0.0, 0.0};
    if (cb == 7) {
      const SlotRec& s = e.slots[c.slot];
      a_lam = s.a_lam;
      if (s.last_corr == k) a_nw = V3{s.a_n[0], s.a_n[1], s.a_n[2]};
    }
    bool ok = true;
    const CorrLin o = correction_linear(e, c, xb, qb, vx, vq, a_lam, a_nw, ok);
    double* Mk = e.cmat + static_cast<size_t>(k % kCorrBatch) * kCorrMat;
    const double col[kCorrRows] = {o.aX.x, o.aX.y, o.aX.z, o.aQ.w, o.aQ.x, o.aQ.y, o.aQ.z,
                                   o.aR.m[0], o.aR.m[1], o.aR.m[2], o.aR.m[3], o.aR.m[4], o.aR.m[5],
                                   o.aR.m[6], o.aR.m[7], o.aR.m[8], o.a_rel.x, o.a_rel.y, o.a_rel.z};
#pragma unroll
    for (int r = 0; r < kCorrRows; ++r) Mk[r * kCorrCols + cb] = col[r];
    if (cb == 7) Mk[kCorrRows * kCorrCols] = ok ? 0.0 : 1.0;
  }
  __syncwarp();
}

// One perturbation simulation (losses.hpp:47-57 with T = 1), forward and,
// when `record`, its adjoint. Returns the residual; status via `status`.
//
// Phase (split execution): kPhaseFused runs forward and adjoint
// in the same warp; kPhaseFwd runs the forward only and stores the state the
// adjoint needs in *rec (its logs stay in the per-(candidate, sim) scratch);
// kPhaseAdj skips the forward, reloads *rec and runs the adjoint.
// One step of a StabilityProtocol with steps > 1 (losses.hpp:54-55): the
// state before the step (prev) and after predict (pred), set by run_sim_steps;
// the forward returns the state after the step, the adjoint takes the adjoint
// of that state and returns the adjoints of pred and of prev's pose (friction's
// "before" point and finalize read prev, sim.hpp:250, 284-285).
__device__ __forceinline__ void put3(double* d, V3 v) { d[0] = v.x; d[1] = v.y; d[2] = v.z; }
__device__ __forceinline__ void put4(double* d, Q4 v) { d[0] = v.w; d[1] = v.x; d[2] = v.y; d[3] = v.z; }
__device__ __forceinline__ V3 get3(const double* d) { return V3{d[0], d[1], d[2]}; }
__device__ __forceinline__ Q4 get4(const double* d) { return Q4{d[0], d[1], d[2], d[3]}; }

struct StepCtx {
  V3 prev_x, prev_xd, prev_w, pred_x, pred_xd, pred_w;
  Q4 prev_q, pred_q;
  // forward out: state after the step, its log sizes
  V3 out_x, out_xd, out_w;
  Q4 out_q;
  int out_ncorr, out_nslot, out_nfric;
  // adjoint in: adjoint of the state after the step
  V3 aX_out, aXd_out, aW_out;
  Q4 aQ_out;
  // adjoint out
  V3 a_pred_x, a_pred_xd, a_pred_w, a_prev_x;
  Q4 a_pred_q, a_prev_q;
};

template <int Phase, class Sdf, bool Multi = false>
__device__ double run_sim(const Sdf& sdf, SimEnv& e, V3 v_m, bool record, bool measure_residual, SimStats& st,
                          int& status, FtAcc& acc, FwdRec* rec, StepCtx* sc = nullptr) {
  const int lane = e.lane, N = e.N;
  // canonical_state (rigid.hpp:29-33) with xdot = v_m; predict (sim.hpp:74-83)
  // (Multi: the step's prev / pred states from run_sim_steps)
  const V3 prev_x = Multi ? sc->prev_x : e.O->com;
  const Q4 prev_q = Multi ? sc->prev_q : Q4{1.0, 0.0, 0.0, 0.0};
  const V3 prev_thd = Multi ? sc->prev_w : V3{0.0, 0.0, 0.0};
  const V3 pred_xdot = Multi ? sc->pred_xd : v_m + V3{0.0 * e.dt, 0.0 * e.dt, 0.0 * e.dt};
  const V3 pred_x = Multi ? sc->pred_x : prev_x + pred_xdot * e.dt;
  const Q4 pred_q = Multi ? sc->pred_q : qnormalized(qmul(quat_exp(prev_thd * e.dt), prev_q));
  // world_inertia_inv at the predicted orientation (sim.hpp:96-100, 142) is
  // KObj::Iw, evaluated once on the host with the same formula (the canonical
  // state has thetadot = 0, so every perturbation predicts the same pose)
  V3 x = pred_x;
  Q4 q = pred_q;
  bool touched = false;
  int ncorr = 0, nslot = 0, nfric = 0;
  const int nwords = (N + 31) / 32;
  if constexpr (Phase == kPhaseAdj || Phase == kPhaseAdjTask) {
    x = V3{rec->x[0], rec->x[1], rec->x[2]};
    q = Q4{rec->q[0], rec->q[1], rec->q[2], rec->q[3]};
    touched = rec->touched != 0;
    ncorr = rec->ncorr;
    nslot = rec->nslot;
    nfric = rec->nfric;
    status = rec->status;
    if (status != kOk) return rec->residual;
  } else {
    M3 R = rotation_matrix(q);
    PoseF Pf{};  // FP32 copy of the pose for the grid pre-filter
    const float radf = static_cast<float>(e.radius);
    if constexpr (kF32Prefilter<Sdf>) Pf = pose_f32(x, R, e.O->com);
    for (int w = lane; w < nwords; w += 32) e.bitmap[w] = 0u;
    if (e.mcert)  // nearest-face certificates are per sim
      for (int i = lane; i < N; i += 32) e.mcert[4 * i + 3] = -1.0;
    __syncwarp();

    PROF_T(tfwd);
    // ---- Gauss-Seidel sweeps (sim.hpp:157-186) -------------------------------
    // Two chunks of 32 consecutive points are classified against the current
    // state (independent straight-line work: ILP); only candidates near /
    // inside the dilated surface run the exact query; the first exact-active
    // point is applied and evaluation restarts right after it. Inactive points
    // change no forward value (sim.hpp:105-125), so this is the sequential sweep.
    int pos = 0, sweep = 0;
    // Quiet window: once N consecutive positions pass with no applied
    // correction (and no singular skip, to keep SolveStats exact), every later
    // position repeats an earlier inactive decision under the same state: the
    // remaining sweeps are skipped. On in the split forward kernel (its other
    // CTA on the SM takes the freed issue slots: 108.2k -> 110.1k); the fused
    // kernel's lockstep CTA measured slower with it, and mesh objects need
    // every point-sweep's (face, sign) cache entry for the adjoint.
    constexpr bool kQuietExit = Phase == kPhaseFwd && !std::is_same<Sdf, MeshSdf>::value;
    int f_last = -1, singular_since = 0;
    while (sweep < e.gs) {
  #if defined(DGX_QUIET) || defined(DGX_QUIET_FWD)  // exact
      if (sweep * N + pos - f_last - 1 >= N && singular_since == 0) break;
  #else
      if constexpr (kQuietExit) {
        if (sweep * N + pos - f_last - 1 >= N && singular_since == 0) break;
      }
  #endif
      // 32-position groups classified per iteration: the split forward kFwdHalves, the fused kernel 2
      // (config 1, fused: 69.3k with 2 groups, 66.8k with 1)
      constexpr int kH = Phase == kPhaseFwd ? kFwdHalves : 2;
      int cls[kH];
  #if DGX_FWD_PREFETCH
      if (e.pts_global) {  // the next chunk's points (global-points forward) into L1 while this one runs
        const int np = pos + 32 * kH < N ? pos + 32 * kH : 0;
  #pragma unroll
        for (int h = 0; h < kH; ++h) {
          const int i = min(np + 32 * h + lane, N - 1);
          asm volatile("prefetch.global.L1 [%0];" ::"l"(e.px + i));
          asm volatile("prefetch.global.L1 [%0];" ::"l"(e.py + i));
          asm volatile("prefetch.global.L1 [%0];" ::"l"(e.pz + i));
        }
      }
  #endif
  #pragma unroll
      for (int h = 0; h < kH; ++h) {
        const int i = pos + 32 * h + lane;
        const int ic = i < N ? i : N - 1;
        if constexpr (kF32Prefilter<Sdf>) {
          // grids: FP32 "certainly inactive" test; everything else -> exact query
          cls[h] = (i >= N || grid_inactive_f32(sdf, Pf, e.px[ic], e.py[ic], e.pz[ic], radf)) ? 1 : 0;
        } else {
          const V3 p{e.px[ic], e.py[ic], e.pz[ic]};
          const V3 rl = ftmul(R, p - x) + e.O->com;
          cls[h] = i < N ? classify_fwd(sdf, e, sweep * N + i, rl).cls : 1;
        }
      }
      unsigned cand[kH];
      unsigned any = 0u;
  #pragma unroll
      for (int h = 0; h < kH; ++h) {
        cand[h] = __ballot_sync(kFull, cls[h] <= 0);
        any |= cand[h];
      }
      PROF_CNT(16, 1);
      if (any == 0u) {
        pos += 32 * kH;
        if (pos >= N) { pos = 0; ++sweep; }
        continue;
      }
      PointEval pe;
      int hsel = -1;
      unsigned mask = 0u;
  #pragma unroll 1
      for (int h = 0; h < kH; ++h) {
        unsigned ch = cand[0];
        int clh = cls[0];
  #pragma unroll
        for (int hh = 1; hh < kH; ++hh)
          if (h == hh) { ch = cand[hh]; clh = cls[hh]; }
        if (ch == 0u) continue;
        const int i = pos + 32 * h + lane;
        bool act = false;
        if (clh <= 0) {
          // grids: R is rebuilt from q here (the same values) instead of being held
          // in registers across the pre-filter loop, which reads only the FP32 pose
          if constexpr (kF32Prefilter<Sdf>) eval_point(sdf, e, i, x, rotation_matrix(q), record, pe);
          else eval_point(sdf, e, i, x, R, record, pe);
          act = record ? (pe.rho_d < 0.0) : !(pe.rho_d >= 0.0);
        }
        mask = __ballot_sync(kFull, act);
        if (mask != 0u) {
          hsel = h;
          break;
        }
      }
      if (hsel < 0) {
        pos += 32 * kH;
        if (pos >= N) { pos = 0; ++sweep; }
        continue;
      }
      const int j = __ffs(mask) - 1;
      const int ij = pos + 32 * hsel + j;
      const V3 rel = shfl(pe.rel, j);
      const V3 g = shfl(pe.q.grad, j);
      const V3 pj = shfl(pe.p, j);
      const double C = -shfl(pe.rho_d, j);
      const V3 dxj = shfl(pe.rl - pe.q.proxy, j);
      const int sgj = __shfl_sync(kFull, pe.q.sign, j);
      const int fbj = __shfl_sync(kFull, pe.fb ? 1 : 0, j);
      // apply_contact (sim.hpp:215-245), out of line (rare path)
      PROF_T(tc);
      const CorrOut co = apply_correction(e, CorrIn{x, q, rel, g, pj, dxj, C, ij, sweep * N + ij, ncorr, nslot, sgj, fbj});
      PROF_ACC(1, tc);
      PROF_CNT(20, 1);
      if (co.status != kOk) { status = co.status; return 0.0; }
      if (co.applied) {
        x = co.x;
        q = co.q;
        if constexpr (kF32Prefilter<Sdf>) Pf = pose_f32(x, rotation_matrix(q), e.O->com);
        else R = rotation_matrix(q);
        touched = true;
        f_last = sweep * N + ij;
        singular_since = 0;
        ++ncorr;
        nslot = co.nslot;
        ++st.corrections;
        st.active += co.new_contact;
      } else {
        ++st.singular;
        ++singular_since;
      }
      pos = ij + 1;
      if (pos >= N) { pos = 0; ++sweep; }
    }

    __syncwarp();  // order the forward's mesh-cache stores before the adjoint's loads
    PROF_ACC(0, tfwd);
    PROF_T(tfr);
    // ---- friction (sim.hpp:188-196), active slots in point order -------------
    if (e.mu > 0.0) {
      for (int wd = 0; wd < nwords; ++wd) {
        unsigned bits = e.bitmap[wd];
        while (bits) {
          const int b = __ffs(bits) - 1;
          bits &= bits - 1u;
          const int pt = wd * 32 + b;
          const int slot = e.slot_of_point[pt];
          const SlotRec& s = e.slots[slot];
          const double lambda_n = s.lambda_n;
          if (lambda_n <= 0.0) continue;
          const V3 x_in = x;
          const Q4 q_in = q;
          Q4 fE{1.0, 0.0, 0.0, 0.0};
          double fsin = 0.0;
          const bool applied =
              friction_fwd(e, prev_x, prev_q, x, q, V3{s.rb[0], s.rb[1], s.rb[2]}, V3{s.n[0], s.n[1], s.n[2]},
                           lambda_n, st, fE, fsin);
          if (applied) {
            touched = true;
            if (lane == 0) {
              SlotRec& sw = e.slots[slot];
              sw.fx[0] = x_in.x; sw.fx[1] = x_in.y; sw.fx[2] = x_in.z;
              sw.fq[0] = q_in.w; sw.fq[1] = q_in.x; sw.fq[2] = q_in.y; sw.fq[3] = q_in.z;
              sw.fE[0] = fE.w; sw.fE[1] = fE.x; sw.fE[2] = fE.y; sw.fE[3] = fE.z;
              sw.fsin = fsin;
              sw.fric = 1;
              e.fric_order[nfric] = slot;
            }
            ++nfric;
            DGX_ASSERT(nfric <= e.slot_cap && slot < e.slot_cap);
          }
          __syncwarp();
        }
      }
    }
    PROF_ACC(2, tfr);
    PROF_CNT(21, nfric);
  }  // forward
  PROF_CNT(22, 1);
  // ---- finalize_velocities (sim.hpp:276-287) and residual ------------------
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
  const double residual = n1 + n2;

  if (measure_residual) {  // sim.hpp:200-208
    M3 Rf = rotation_matrix(q);
    double mp = 0.0;
    for (int i = lane; i < N; i += 32) {
      V3 p{e.px[i], e.py[i], e.pz[i]};
      V3 rl = tmul(Rf, p - x) + e.O->com;
      if (sdf_culled(sdf, rl, e.radius)) continue;  // sim.hpp:204-205
      SdfQuery qq = sdf.query(rl);
      double rho = qq.rho - e.radius;
      if (rho < 0.0) mp = mp < -rho ? -rho : mp;
    }
    const double wm = warp_max(mp);
    st.max_pen = Multi ? (st.max_pen < wm ? wm : st.max_pen) : wm;  // one SolveStats over the steps
  }
  if constexpr (Multi && Phase == kPhaseFwd) {
    sc->out_x = x;
    sc->out_q = q;
    sc->out_xd = xdot;
    sc->out_w = thd;
    sc->out_ncorr = ncorr;
    sc->out_nslot = nslot;
    sc->out_nfric = nfric;
  }
  if constexpr (Phase == kPhaseFwd) {  // the adjoint kernel resumes from here
    if (lane == 0) {
      rec->x[0] = x.x; rec->x[1] = x.y; rec->x[2] = x.z;
      rec->q[0] = q.w; rec->q[1] = q.x; rec->q[2] = q.y; rec->q[3] = q.z;
      rec->touched = touched ? 1 : 0;
      rec->ncorr = ncorr;
      rec->nslot = nslot;
      rec->nfric = nfric;
    }
    return residual;
  }
  V3 aX;
  Q4 aQ;
  if constexpr (Multi) {
    // finalize (sim.hpp:276-287) reverse with the adjoint of the step's output
    sc->a_pred_xd = V3{0.0, 0.0, 0.0};
    sc->a_pred_w = V3{0.0, 0.0, 0.0};
    sc->a_prev_x = V3{0.0, 0.0, 0.0};
    sc->a_prev_q = Q4{0.0, 0.0, 0.0, 0.0};
    aX = sc->aX_out;
    aQ = sc->aQ_out;
    if (!touched) {  // xdot / thetadot pass through from predict; x / q carry only the leak
      sc->a_pred_xd = sc->aXd_out;
      sc->a_pred_w = sc->aW_out;
    } else {
      const Q4 a_qd = quat_log_adj(qd, sc->aW_out * inv_dt);
      aQ = qadd(aQ, qmul_adj_a(a_qd, qconj(prev_q)));
      const Q4 ac = qmul_adj_b(a_qd, q);
      sc->a_prev_q = Q4{ac.w, -ac.x, -ac.y, -ac.z};
      aX = aX + sc->aXd_out * inv_dt;
      sc->a_prev_x = sc->aXd_out * -inv_dt;
    }
    const bool zero = aX.x == 0.0 && aX.y == 0.0 && aX.z == 0.0 && aQ.w == 0.0 && aQ.x == 0.0 && aQ.y == 0.0 &&
                      aQ.z == 0.0;
    sc->a_pred_x = aX;
    sc->a_pred_q = aQ;
    if (!record || zero) return residual;  // the tape skips zero adjoints (tape.cpp:33)
  } else {
    if (!record || !touched) return residual;  // untouched: constant loss, zero gradient
  }
  PROF_CNT(32, 1);
  PROF_CNT(36, ncorr);

  for (int t = lane; t < 6 * e.L; t += 32) e.gft[t] = 0.0;
  __syncwarp();
  // ---- adjoint: residual -> finalize ---------------------------------------
  if constexpr (!Multi) {
    const V3 a_xdot = n1 > 0.0 ? xdot / n1 : V3{0.0, 0.0, 0.0};
    const V3 a_thd = n2 > 0.0 ? thd / n2 : V3{0.0, 0.0, 0.0};
    aQ = qmul_adj_a(quat_log_adj(qd, a_thd * inv_dt), qconj(prev_q));
    aX = a_xdot * inv_dt;
  }

  PROF_T(tfa);
  // ---- friction, reverse --------------------------------------------------
  // Each friction's reverse step is linear in v = (aX, aQ) given its logged
  // forward values: v <- A_k v, a_lam_k = l_k . v, a_n_k = N_k v (11 x 7).
  // Batches of frictions get their matrices in parallel (one lane per
  // friction, friction_adj on the 7 basis vectors, staged in shared memory);
  // the serial chain is then one 11 x 7 mat-vec per friction (lanes = rows)
  // instead of one full reverse step.
  {
    constexpr int kFr = 11 * 7;
    const int nb_max = min(32, (e.seg_max * 5 * 32) / kFr);
    int hi = nfric;
    while (hi > 0) {
      const int cnt = (!Multi && nb_max >= 2) ? min(nb_max, hi) : 1;
      if (cnt == 1) {  // serial reverse step (short tails / tiny staging; Multi: with prev's adjoint)
        const int slot = e.fric_order[hi - 1];
        SlotRec s = e.slots[slot];
        double a_lam = s.a_lam;
        V3 a_n{s.a_n[0], s.a_n[1], s.a_n[2]};
        friction_adj(e, prev_x, prev_q, s, aX, aQ, a_lam, a_n, Multi ? &sc->a_prev_x : nullptr,
                     Multi ? &sc->a_prev_q : nullptr);
        __syncwarp();
        if (lane == 0) {
          SlotRec& sw = e.slots[slot];
          sw.a_lam = a_lam;
          sw.a_n[0] = a_n.x; sw.a_n[1] = a_n.y; sw.a_n[2] = a_n.z;
        }
        __syncwarp();
        --hi;
        continue;
      }
      if (lane < cnt) {  // lane j: friction hi - 1 - j
        const SlotRec s = e.slots[e.fric_order[hi - 1 - lane]];
        double* Mj = e.stage + lane * kFr;
#pragma unroll 1
        for (int c = 0; c < 7; ++c) {
          V3 bx{c == 0 ? 1.0 : 0.0, c == 1 ? 1.0 : 0.0, c == 2 ? 1.0 : 0.0};
          Q4 bq{c == 3 ? 1.0 : 0.0, c == 4 ? 1.0 : 0.0, c == 5 ? 1.0 : 0.0, c == 6 ? 1.0 : 0.0};
          double al = 0.0;
          V3 an{0.0, 0.0, 0.0};
          friction_adj(e, prev_x, prev_q, s, bx, bq, al, an);
          const double col[11] = {bx.x, bx.y, bx.z, bq.w, bq.x, bq.y, bq.z, al, an.x, an.y, an.z};
#pragma unroll
          for (int r = 0; r < 11; ++r) Mj[r * 7 + c] = col[r];
        }
      }
      __syncwarp();
      for (int j = 0; j < cnt; ++j) {
        const double v[7] = {aX.x, aX.y, aX.z, aQ.w, aQ.x, aQ.y, aQ.z};
        double r = 0.0;
        if (lane < 11) {
          const double* row = e.stage + j * kFr + lane * 7;
#pragma unroll
          for (int c = 0; c < 7; ++c) r = fma(row[c], v[c], r);
        }
        aX = V3{shfl(r, 0), shfl(r, 1), shfl(r, 2)};
        aQ = Q4{shfl(r, 3), shfl(r, 4), shfl(r, 5), shfl(r, 6)};
        const double al = shfl(r, 7);
        const V3 an{shfl(r, 8), shfl(r, 9), shfl(r, 10)};
        if (lane == 0) {
          SlotRec& sw = e.slots[e.fric_order[hi - 1 - j]];
          sw.a_lam = sw.a_lam + al;
          sw.a_n[0] = sw.a_n[0] + an.x; sw.a_n[1] = sw.a_n[1] + an.y; sw.a_n[2] = sw.a_n[2] + an.z;
        }
      }
      __syncwarp();
      hi -= cnt;
    }
  }

  PROF_ACC(4, tfa);
  PROF_T(tcm);
  int built_lo = ncorr;  // matrices of corrections [built_lo, ...] are in the ring
  PROF_ACC(11, tcm);
  // ---- sweeps, reverse ----------------------------------------------------
  M3 aR;  // per-lane partial adjoint of the current R node
  for (int k = 0; k < 9; ++k) aR.m[k] = 0.0;
  // Reverse sweep as a state machine with ONE process_run call site (keeps
  // the i-cache footprint of the inlined adjoint small):
  //   stage 0/1/2 fold the final run [lo_f, hi): the last correction is
  //     followed by K >= 2 identical cycles of the same N point-sweeps with the
  //     same state (plus a partial head of r positions). Stage 0 processes the
  //     head; stage 1 runs ONE cycle in map-only mode (its affine map
  //     a -> M a + b on adj_x); the adjoint is iterated K times through it;
  //     stage 2 runs one emission pass fed sum_k X_k with c0 scaled by K, which
  //     emits all K cycles by linearity.
  //   stage 3 walks the remaining runs and logged corrections in reverse.
  int hi = e.gs * N;
  const int lo_f = ncorr > 0 ? e.corr[ncorr - 1].f + 1 : 0;
  const int Kc = (hi - lo_f) / N;
  const int rhead = (hi - lo_f) - Kc * N;
  PROF_CNT(33, Kc >= 2 ? 1 : 0);
  PROF_CNT(34, Kc);
#ifdef DGX_QUIET
  int stage = Kc >= 2 ? 0 : 3;
#else
  // the warp-task adjoint folds (its warps do not wait on each other, so the
  // saved work is not lost to a barrier); DESIGN.md §3
  // (the CTA-per-candidate adjoint measured slower with it: its warps wait at
  // the candidate barrier, and the fold's code alone costs it issue slots)
  int stage = (Phase == kPhaseAdjTask && e.fold && Kc >= 2) ? 0 : 3;
#endif
  int k = ncorr - 1;
  V3 Xk_fold{0.0, 0.0, 0.0};
  M3 Mc;
  V3 bc{0.0, 0.0, 0.0};
  for (;;) {
    const int kstate = stage < 3 ? ncorr - 1 : k;  // state after correction kstate
    V3 xk = pred_x;
    Q4 qk = pred_q;
    if (kstate >= 0) {
      const CorrRec& c = e.corr[kstate];
      xk = V3{c.x[0], c.x[1], c.x[2]};
      qk = Q4{c.q[0], c.q[1], c.q[2], c.q[3]};
    }
    const M3 Rk = rotation_matrix(qk);
    int lo = 0, hr = 0;
    double scale = 1.0;
    bool mapm = false;
    if (stage == 0) {
      lo = hi - rhead;
      hr = hi;
    } else if (stage == 1 || stage == 2) {
      lo = lo_f;
      hr = lo_f + N;
      mapm = stage == 1;
      scale = stage == 2 ? static_cast<double>(Kc) : 1.0;
    } else {
      lo = k >= 0 ? e.corr[k].f + 1 : 0;
      hr = hi;
    }
    V3 aXrun = aX;
    PROF_T(tpr);
    process_run(sdf, e, lo, hr, xk, qk, Rk, aQ, aXrun, aR, acc, scale, mapm ? &Mc : nullptr, mapm ? &bc : nullptr);
    PROF_ACC(5, tpr);
    PROF_CNT(19, 1);
    if (stage == 0) {
      aX = aXrun;
      stage = 1;
      continue;
    }
    if (stage == 1) {
      V3 Y{0.0, 0.0, 0.0};
      Xk_fold = aX;
      for (int j = 0; j < Kc; ++j) {
        Y = Y + Xk_fold;
        Xk_fold = fmul(Mc, Xk_fold) + bc;
      }
      aX = Y;  // input of the emission pass
      stage = 2;
      continue;
    }
    if (stage == 2) {
      aX = Xk_fold;  // adjoint entering the final run from below
      hi = lo_f;
      stage = 3;
      continue;
    }
    aX = aXrun;
    if (k < 0) break;

    // ---- active correction k (sim.hpp:215-245), reverse ----
    PROF_T(tca);
    const M3 aRk = warp_sum(aR);
    aQ = qadd(aQ, rotmat_adj(qk, aRk));
    for (int t = 0; t < 9; ++t) aR.m[t] = 0.0;
    if (k < built_lo) {  // next batch of correction matrices, built in parallel
      built_lo = max(0, k - kCorrBatch + 1);
      correction_matrices(e, built_lo, k, pred_x, pred_q);
    }
    {  // the precomputed affine map of correction k: one 19 x 8 mat-vec (lanes = rows)
      const double* Mk = e.cmat + static_cast<size_t>(k % kCorrBatch) * kCorrMat;
      const double v[kCorrCols] = {aX.x, aX.y, aX.z, aQ.w, aQ.x, aQ.y, aQ.z, 1.0};
      double r = 0.0;
      if (lane < kCorrRows) {
        const double* row = Mk + lane * kCorrCols;
#pragma unroll
        for (int c = 0; c < kCorrCols; ++c) r = fma(row[c], v[c], r);
      }
      aX = V3{shfl(r, 0), shfl(r, 1), shfl(r, 2)};
      aQ = Q4{shfl(r, 3), shfl(r, 4), shfl(r, 5), shfl(r, 6)};
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        const double m = shfl(r, 7 + t);
        aR.m[t] = lane == 0 ? m : 0.0;
      }
      const V3 a_rel{shfl(r, 16), shfl(r, 17), shfl(r, 18)};
      if (lane == 0) {
        if (Mk[kCorrRows * kCorrCols] != 0.0) status = kReplayMismatch;
        const int i = e.corr[k].f % e.N;
        const V3 p{e.px[i], e.py[i], e.pz[i]};
        double* d = e.ft + 6 * e.sample_link[i];
        const V3 tq = cross(p, a_rel);
        d[0] += a_rel.x; d[1] += a_rel.y; d[2] += a_rel.z;
        d[3] += tq.x; d[4] += tq.y; d[5] += tq.z;
        add_point_grad(e, i, a_rel);
      }
      __syncwarp();
    }
    PROF_ACC(11, tca);
    hi = e.corr[k].f;
    --k;
  }
  if constexpr (Multi) {  // the sweeps started from pred (st = predicted, sim.hpp:144)
    // the solve's first R node, rotation_matrix(pred.theta) (sim.hpp:145), read
    // by the run before the first correction (a constant when T = 1)
    aQ = qadd(aQ, rotmat_adj(pred_q, warp_sum(aR)));
    sc->a_pred_x = aX;
    sc->a_pred_q = aQ;
  }
  // fold the global spill buffer into the warp's shared link sums
  PROF_T(tf);
  acc.spill_if_any(e.gft);
  __threadfence();
  __syncwarp();
  for (int t = lane; t < 6 * e.L; t += 32) e.ft[t] += __ldcg(e.gft + t);
  __syncwarp();
  PROF_ACC(10, tf);
  if (e.discard) {  // this sim's logs and correction matrices are consumed
    l2_discard(e.cmat, static_cast<size_t>(min(ncorr, kCorrBatch)) * kCorrMat * sizeof(double), lane, 32);
    l2_discard(e.corr, static_cast<size_t>(ncorr) * sizeof(CorrRec), lane, 32);
    l2_discard(e.slots, static_cast<size_t>(nslot) * sizeof(SlotRec), lane, 32);
  }
  return residual;
}



// perturbation_residual with StabilityProtocol::steps = T > 1 (losses.hpp:47-57):
// T steps of predict + solve (sim.hpp:310-316) from the canonical state, the
// residual of the last, and (record) the reverse over the steps: each step's
// adjoint (run_sim<kPhaseAdj, Multi>) followed by predict's reverse
// (sim.hpp:74-83: pred.x = x + dt pred.xdot, pred.theta = normalized(
// quat_exp(dt thetadot) (x) theta)). The world inverse inertia is frozen per
// step at its predicted orientation (sim.hpp:142). Logs of all T solves are
// kept (corrections / slots / frictions at per-step offsets); link sums
// accumulate over the steps (the hand points are shared).
template <class Sdf>
__device__ double run_sim_steps(const Sdf& sdf, SimEnv& e, V3 v_m, bool record, bool meas, SimStats& st,
                                int& status, FtAcc& acc, StepRec* steps, int T) {
  const int lane = e.lane;
  CorrRec* corr0 = e.corr;
  SlotRec* slots0 = e.slots;
  int* fo0 = e.fric_order;
  int* mc0 = e.mcache;
  const int cap0 = e.cap_corr, scap0 = e.slot_cap;
  const KObj* O0 = e.O;
  KObj Ot = *O0;  // Iw at each step's predicted orientation
  e.O = &Ot;
  auto bind_step = [&](int c_off, int s_off, int f_off, int t) {
    e.corr = corr0 + c_off;
    e.slots = slots0 + s_off;
    e.fric_order = fo0 + f_off;
    e.cap_corr = cap0 - c_off;
    e.slot_cap = scap0 - s_off;
    if (mc0) e.mcache = mc0 + static_cast<size_t>(t) * e.gs * e.N;
  };
  auto set_iw = [&](Q4 pq) {
    const M3 Rp = rotation_matrix(pq);
    Ot.Iw = mul(mul(Rp, O0->inertia_body_inv), transposed(Rp));  // sim.hpp:96-100
  };
  V3 x = O0->com, xd = v_m, w{0.0, 0.0, 0.0};  // canonical_state with xdot = v (losses.hpp:52-53)
  Q4 q{1.0, 0.0, 0.0, 0.0};
  int c_off = 0, s_off = 0, f_off = 0;
  double residual = 0.0;
  for (int t = 0; t < T; ++t) {
    StepCtx sc;
    sc.prev_x = x; sc.prev_q = q; sc.prev_xd = xd; sc.prev_w = w;
    sc.pred_xd = xd + V3{0.0 * e.dt, 0.0 * e.dt, 0.0 * e.dt};  // gravity zeroed (losses.hpp:51)
    sc.pred_x = x + sc.pred_xd * e.dt;
    sc.pred_q = qnormalized(qmul(quat_exp(w * e.dt), q));
    sc.pred_w = w;
    set_iw(sc.pred_q);
    bind_step(c_off, s_off, f_off, t);
    StepRec& sr = steps[t];
    residual = run_sim<kPhaseFwd, Sdf, true>(sdf, e, v_m, record, meas, st, status, acc, &sr.rec, &sc);
    if (lane == 0) {
      sr.rec.status = status;
      sr.rec.residual = residual;
      put3(sr.prev, x); put4(sr.prev + 3, q); put3(sr.prev + 7, xd); put3(sr.prev + 10, w);
      put3(sr.pred, sc.pred_x); put4(sr.pred + 3, sc.pred_q); put3(sr.pred + 7, sc.pred_xd); put3(sr.pred + 10, sc.pred_w);
      sr.c_off = c_off; sr.s_off = s_off; sr.f_off = f_off;
    }
    __syncwarp();
    if (status != kOk) {
      e.O = O0;
      return residual;
    }
    c_off += sc.out_ncorr;
    s_off += sc.out_nslot;
    f_off += sc.out_nfric;
    x = sc.out_x; q = sc.out_q; xd = sc.out_xd; w = sc.out_w;
  }
  if (record) {
    const double n1 = norm(xd), n2 = norm(w);
    V3 aX{0.0, 0.0, 0.0}, aXd = n1 > 0.0 ? xd / n1 : V3{0.0, 0.0, 0.0}, aW = n2 > 0.0 ? w / n2 : V3{0.0, 0.0, 0.0};
    Q4 aQ{0.0, 0.0, 0.0, 0.0};
    for (int t = T - 1; t >= 0; --t) {
      const StepRec& sr = steps[t];
      StepCtx sc;
      sc.prev_x = get3(sr.prev); sc.prev_q = get4(sr.prev + 3); sc.prev_xd = get3(sr.prev + 7); sc.prev_w = get3(sr.prev + 10);
      sc.pred_x = get3(sr.pred); sc.pred_q = get4(sr.pred + 3); sc.pred_xd = get3(sr.pred + 7); sc.pred_w = get3(sr.pred + 10);
      sc.aX_out = aX; sc.aQ_out = aQ; sc.aXd_out = aXd; sc.aW_out = aW;
      set_iw(sc.pred_q);
      bind_step(sr.c_off, sr.s_off, sr.f_off, t);
      SimStats st2;
      int s2 = kOk;
      run_sim<kPhaseAdj, Sdf, true>(sdf, e, v_m, true, false, st2, s2, acc, const_cast<FwdRec*>(&sr.rec), &sc);
      if (s2 != kOk) status = s2;
      // predict, reverse (sim.hpp:74-83)
      aXd = fma3(e.dt, sc.a_pred_x, sc.a_pred_xd);
      aX = sc.a_pred_x + sc.a_prev_x;
      double sh;
      const Q4 E = quat_exp_sin(sc.prev_w * e.dt, sh);
      const Q4 aP = qnormalize_adj(qmul(E, sc.prev_q), sc.a_pred_q);
      aQ = qadd(qmul_adj_b(aP, E), sc.a_prev_q);
      const V3 aom = quat_exp_adj_sc(sc.prev_w * e.dt, qmul_adj_a(aP, sc.prev_q), sh, E.w);
      aW = fma3(e.dt, aom, sc.a_pred_w);
    }
  }
  e.O = O0;
  e.corr = corr0;
  e.slots = slots0;
  e.fric_order = fo0;
  e.cap_corr = cap0;
  e.slot_cap = scap0;
  e.mcache = mc0;
  return residual;
}

// HandModel::forward (hand.hpp:116-152) link transforms, lane 0 serial over
// the BFS order. base_q is the recorded orientation quat_exp(0) (x) q0
// (hand.cpp:250-253) on the recorded path, q0 itself on the forward path.
__device__ __forceinline__ void link_transforms(const KHand& H, const double* qv, bool record, double* link) {
  Q4 q0{qv[3], qv[4], qv[5], qv[6]};
  Q4 base_q = record ? qmul(quat_exp(V3{0.0, 0.0, 0.0}), q0) : q0;
  for (int k = 0; k < H.L; ++k) {
    const int li = H.topo[k];
    double* Rl = link + 12 * li;
    const int pj = H.link_parent_joint[li];
    M3 R;
    V3 t;
    if (pj < 0) {
      R = rotation_matrix(base_q);
      t = V3{qv[0], qv[1], qv[2]};
    } else {
      const double angle = qv[7 + pj];
      const V3 ax{H.axis[3 * pj], H.axis[3 * pj + 1], H.axis[3 * pj + 2]};
      const V3 rotvec{ax.x * angle, ax.y * angle, ax.z * angle};
      const M3 Rj = rotation_matrix(quat_exp(rotvec));
      M3 Ro;
      for (int m = 0; m < 9; ++m) Ro.m[m] = H.origin_R[9 * pj + m];
      const V3 to{H.origin_t[3 * pj], H.origin_t[3 * pj + 1], H.origin_t[3 * pj + 2]};
      const double* Pp = link + 12 * H.joint_parent[pj];
      M3 Rp;
      for (int m = 0; m < 9; ++m) Rp.m[m] = Pp[m];
      const V3 tp{Pp[9], Pp[10], Pp[11]};
      R = mul(mul(Rp, Ro), Rj);
      t = mul(Rp, to) + tp;
    }
    for (int m = 0; m < 9; ++m) Rl[m] = R.m[m];
    Rl[9] = t.x; Rl[10] = t.y; Rl[11] = t.z;
  }
}

// link_transforms by one warp (lane k: link topo[k]; L <= 27). The joint
// rotations quat_exp(axis * angle) do not depend on the parent and are built
// by all lanes at once; the products R_parent * R_origin * R_joint then go
// level by level (a link as soon as its parent is done). Every link's values
// are the same operations as link_transforms, so the results are identical.
__device__ __forceinline__ void link_transforms_warp(const KHand& H, const double* qv, bool record, double* link,
                                                     int lane) {
  const bool mine = lane < H.L;
  const int li = mine ? H.topo[lane] : 0;
  const int pj = mine ? H.link_parent_joint[li] : -1;
  int kpar = -1;  // topo index of the parent link
  M3 Rj;
  if (mine && pj >= 0) {
    const int pl = H.joint_parent[pj];
    for (int k = 0; k < H.L; ++k)
      if (H.topo[k] == pl) kpar = k;
    const double angle = qv[7 + pj];
    const V3 ax{H.axis[3 * pj], H.axis[3 * pj + 1], H.axis[3 * pj + 2]};
    const V3 rotvec{ax.x * angle, ax.y * angle, ax.z * angle};
    Rj = rotation_matrix(quat_exp(rotvec));
  }
  const unsigned all = H.L >= 32 ? kFull : ((1u << H.L) - 1u);
  unsigned done = 0u;
  while (done != all) {
    const bool ready = mine && !((done >> lane) & 1u) && (pj < 0 || ((done >> kpar) & 1u));
    if (ready) {
      double* Rl = link + 12 * li;
      M3 R;
      V3 t;
      if (pj < 0) {
        const Q4 q0{qv[3], qv[4], qv[5], qv[6]};
        const Q4 base_q = record ? qmul(quat_exp(V3{0.0, 0.0, 0.0}), q0) : q0;
        R = rotation_matrix(base_q);
        t = V3{qv[0], qv[1], qv[2]};
      } else {
        M3 Ro;
        for (int m = 0; m < 9; ++m) Ro.m[m] = H.origin_R[9 * pj + m];
        const V3 to{H.origin_t[3 * pj], H.origin_t[3 * pj + 1], H.origin_t[3 * pj + 2]};
        const double* Pp = link + 12 * H.joint_parent[pj];
        M3 Rp;
        for (int m = 0; m < 9; ++m) Rp.m[m] = Pp[m];
        const V3 tp{Pp[9], Pp[10], Pp[11]};
        R = mul(mul(Rp, Ro), Rj);
        t = mul(Rp, to) + tp;
      }
      for (int m = 0; m < 9; ++m) Rl[m] = R.m[m];
      Rl[9] = t.x; Rl[10] = t.y; Rl[11] = t.z;
    }
    __syncwarp();
    done |= __ballot_sync(kFull, ready);
  }
}

// FK adjoint: link force/torque sums -> gradient [pos | tangent | joints]
// (hand.cpp:246-257 layout). ft is consumed (subtree sums in place). Called by
// a whole warp: lane 0 folds the subtrees in reverse topo order (the sums'
// order is fixed), then lanes take one joint each.
__device__ __forceinline__ void fk_adjoint(const KHand& H, const double* qv, const double* link, double* ft, double* g,
                                           int lane) {
  if (lane == 0) {
    for (int k = H.L - 1; k >= 1; --k) {
      const int li = H.topo[k];
      const int par = H.joint_parent[H.link_parent_joint[li]];
      for (int c = 0; c < 6; ++c) ft[6 * par + c] += ft[6 * li + c];
    }
    const int base = H.topo[0];
    const V3 F{ft[6 * base], ft[6 * base + 1], ft[6 * base + 2]};
    const V3 T{ft[6 * base + 3], ft[6 * base + 4], ft[6 * base + 5]};
    const V3 pos{qv[0], qv[1], qv[2]};
    const V3 tau = (F.x == 0.0 && F.y == 0.0 && F.z == 0.0) ? T : T - cross(pos, F);
    g[0] = F.x; g[1] = F.y; g[2] = F.z;
    g[3] = tau.x; g[4] = tau.y; g[5] = tau.z;
  }
  __syncwarp();
  for (int j = lane; j < H.J; j += 32) {
    const int c = H.joint_child[j], p = H.joint_parent[j];
    // the tape never propagates a zero adjoint (tape.cpp:33): a subtree without
    // adjoint contributes exactly 0 even where pose values are non-finite
    bool zero = true;
    for (int t = 0; t < 6; ++t) zero = zero && ft[6 * c + t] == 0.0;
    if (zero) {
      g[6 + j] = 0.0;
      continue;
    }
    M3 Rp, Ro;
    for (int m = 0; m < 9; ++m) { Rp.m[m] = link[12 * p + m]; Ro.m[m] = H.origin_R[9 * j + m]; }
    const V3 aw = mul(Rp, mul(Ro, V3{H.axis[3 * j], H.axis[3 * j + 1], H.axis[3 * j + 2]}));
    const V3 tc{link[12 * c + 9], link[12 * c + 10], link[12 * c + 11]};
    const V3 Fc{ft[6 * c], ft[6 * c + 1], ft[6 * c + 2]};
    const V3 Tc{ft[6 * c + 3], ft[6 * c + 4], ft[6 * c + 5]};
    g[6 + j] = dot(aw, Tc - cross(tc, Fc));
  }
  __syncwarp();
}

// CTAs per SM the register budget is sized for: mesh objects spend ~99% of
// the time in out-of-line BVH traversals (latency-bound), so their instance
// trades adjoint-side spills for a second resident CTA
template <class Sdf>
struct CtasPerSm {
  static constexpr int value = 1;
};
template <>
struct CtasPerSm<MeshSdf> {
  static constexpr int value = 2;
};

// Split-execution forward kernel: 2 CTAs per SM (the adjoint is compiled out
// of this instance). Config 2: 2 CTAs/SM 101k cand-iter/s, 3 CTAs/SM (80
// registers, 1 KB of spills) 96k, fused 86k.
#ifndef DGX_FWD_CTAS
#define DGX_FWD_CTAS 2
#endif
constexpr int kFwdCtasPerSm = DGX_FWD_CTAS;
// the global-points forward (large hands: 24 KB of shared memory per CTA) at 5
// CTAs per SM: config 3 forward with one 32-position group per iteration
// 4 / 5 / 6 / 7 CTAs 15.26 / 14.73 / 19.7 / 30.0 ms per step (5: 56 registers,
// 1.3 KB of spills; with two groups 2 / 3 / 4 / 5 CTAs 17.2 / 16.8 / 15.6 /
// 16.5 ms); with the points in shared memory 3 CTAs lose (config 2 1.40 ->
// 1.86 ms, config 4 2.48 -> 3.03 ms)
#ifndef DGX_FWD_CTAS_PTSG
#define DGX_FWD_CTAS_PTSG 5
#endif
constexpr int kFwdCtasPerSmPtsG = DGX_FWD_CTAS_PTSG;
// the forward's SDF parameter stays a by-value copy (measured: as a
// __grid_constant__ parameter the config-3 forward ran 17.5 -> 18.0 ms); the
// other structs and the other kernels' parameters are __grid_constant__ (no
// local copies: config-3 lane adjoint 29.1 -> 28.2 ms)
#ifndef DGX_FWD_SDF_GC
#define DGX_FWD_SDF_GC
#endif

// The CTA's next candidate after b. Candidates differ in cost (contacts,
// corrections), so a CTA that finishes early takes the next unclaimed one
// instead of its static stride. Per-candidate math does not depend on which
// CTA runs it (split: logs per candidate; fused: per-CTA scratch is rebound
// each candidate), so results are identical to the static schedule.
// s_next: a dynamic shared-memory slot (static shared memory would push the
// kernels' 227 KB dynamic opt-in over the per-CTA limit).
__device__ __forceinline__ int next_candidate(const KBuf& buf, int b, int* s_next) {
  if (buf.claim == nullptr) return b + gridDim.x;
  __syncthreads();  // every thread has read the previous claim
  if (threadIdx.x == 0)
    *s_next = static_cast<int>(min(atomicAdd(buf.claim, 1ull), static_cast<unsigned long long>(INT_MAX / 2))) +
              static_cast<int>(gridDim.x);
  __syncthreads();
  return *s_next;
}

// Per-candidate epilogue of one candidate-iteration, by one warp (losses.cpp:
// 20-66 reductions, qrange / qlimit losses.hpp:70-93, the FK adjoint, and for
// the optimizer App. C: weighted gradient, Adam, apply_gradient_step
// losses.cpp:92-102). sflag / sres: per-sim status and residuals [M]; ft_all:
// per-sim link sums [M][6L] (summed per entry in sim order); scratch: >= 6L
// doubles; sg: [3*32]; sq: the configuration (updated in place by a step).
// Shared by the CTA-per-candidate kernels and the warp-task adjoint.
__device__ __forceinline__ void candidate_epilogue(const KHand& H, const KSim& S, const KOpt& P, const KBuf& buf,
                                                   int mode, int b, int k, int lane, const int* sflag,
                                                   const double* sres, const double* ft_all, const double* link,
                                                   double* scratch, double* sg, double* sq, double& am, double& av,
                                                   double& b1t, double& b2t, int& cand_status) {
  const int M = S.M, L = H.L, J = H.J, D = 6 + J;
  const bool record = mode != kModeEval;
  double* stage_all = scratch;
  for (int m = 0; m < M; ++m)
    if (sflag[m] != kOk) cand_status = sflag[m];
  // stability loss: losses.cpp:43-45 (record) / losses.hpp:60-67 (eval)
  double stable = 0.0;
  for (int m = 0; m < M; ++m) stable = stable + sres[m];
  if (record) stable = stable * (1.0 / static_cast<double>(M));
  else stable = stable / static_cast<double>(M);
  // qrange / qlimit (losses.hpp:70-93)
  double qr = 0.0, ql = 0.0;
  for (int j = 0; j < J; ++j) {
    const double d = sq[7 + j] - 0.5 * (H.lower[j] + H.upper[j]);
    qr = qr + d * d;
  }
  qr = sqrt(qr);
  for (int j = 0; j < J; ++j) {
    const double a = sq[7 + j] - H.upper[j];
    ql = ql + (a >= 0.0 ? a : 0.0);
    const double c = H.lower[j] - sq[7 + j];
    ql = ql + (c >= 0.0 ? c : 0.0);
  }
  if (record) {
    // link sums over the sims (losses.cpp:32-41 order, per entry), lanes over entries
    for (int t = lane; t < 6 * L; t += 32) {
      double s = 0.0;
      for (int m = 0; m < M; ++m) s += ft_all[m * 6 * L + t];
      stage_all[t] = s;
    }
    __syncwarp();
    fk_adjoint(H, sq, link, stage_all, sg, lane);
    __syncwarp();
    if (lane < D) {
      const double inv_m = 1.0 / static_cast<double>(M);
      double ds = sg[lane] * inv_m;
      double dr = 0.0, dl = 0.0;
      if (lane >= 6) {
        const int j = lane - 6;
        const double d = sq[7 + j] - 0.5 * (H.lower[j] + H.upper[j]);
        dr = qr > 0.0 ? 2.0 * ((0.5 / qr) * d) : 0.0;
        dl = (sq[7 + j] - H.upper[j] >= 0.0 ? 1.0 : 0.0) + (H.lower[j] - sq[7 + j] >= 0.0 ? -1.0 : 0.0);
      }
      sg[lane] = ds;
      sg[32 + lane] = dr;
      sg[64 + lane] = dl;
    }
    __syncwarp();
  }
  const bool finite_loss = isfinite(stable) && isfinite(qr) && isfinite(ql);
  if (!finite_loss && cand_status == kOk) cand_status = kNonFiniteLoss;
  if (mode == kModeGrad || mode == kModeEval) {
    if (lane == 0 && buf.losses) {
      double* lo = buf.losses + static_cast<size_t>(b) * 3;
      lo[0] = stable; lo[1] = qr; lo[2] = ql;
    }
    if (mode == kModeGrad && lane < D && buf.grads) {
      double* go = buf.grads + static_cast<size_t>(b) * 3 * D;
      go[lane] = sg[lane];
      go[D + lane] = sg[32 + lane];
      go[2 * D + lane] = sg[64 + lane];
      if (!isfinite(sg[lane]) && cand_status == kOk) cand_status = kNonFiniteGrad;
    }
  } else {
    // App. C: weighted gradient, Adam, apply_gradient_step
    double gw = 0.0;
    if (lane < D) gw = S.w_stable * sg[lane] + S.w_qrange * sg[32 + lane] + S.w_qlimit * sg[64 + lane];
    if (buf.egrad && lane < D) gw = gw + buf.egrad[static_cast<size_t>(b) * D + lane];  // grasp energies
    const bool bad = __any_sync(kFull, lane < D && !isfinite(gw));
    if (bad && cand_status == kOk) cand_status = kNonFiniteGrad;
    if (buf.traj) {
      double* tr = buf.traj + (static_cast<size_t>(b) * P.traj_rows + (k - P.traj_k0)) * (3 + D);
      if (lane == 0) { tr[0] = stable; tr[1] = qr; tr[2] = ql; }
      if (lane < D) tr[3 + lane] = gw;
    }
    b1t = b1t * P.beta1;
    b2t = b2t * P.beta2;
    double dir = 0.0;
    if (lane < D) {
      const double c1 = 1.0 - P.beta1, c2 = 1.0 - P.beta2;
      am = P.beta1 * am + c1 * gw;
      av = P.beta2 * av + c2 * (gw * gw);
      const double mhat = am / (1.0 - b1t);
      const double vhat = av / (1.0 - b2t);
      dir = mhat / (sqrt(vhat) + P.eps);
    }
    __syncwarp();
    if (lane < D) sg[lane] = dir;  // sg now holds the step direction
    __syncwarp();
    if (lane == 0 && cand_status == kOk) {
      // apply_gradient_step (losses.cpp:92-102)
      const double lr = P.lr;
      sq[0] = sq[0] - lr * sg[0];
      sq[1] = sq[1] - lr * sg[1];
      sq[2] = sq[2] - lr * sg[2];
      const V3 tangent{-lr * sg[3], -lr * sg[4], -lr * sg[5]};
      const Q4 qn = qnormalized(qmul(quat_exp(tangent), Q4{sq[3], sq[4], sq[5], sq[6]}));
      sq[3] = qn.w; sq[4] = qn.x; sq[5] = qn.y; sq[6] = qn.z;
      for (int j = 0; j < J; ++j) sq[7 + j] = sq[7 + j] - lr * sg[6 + j];
    }
  }
}

// PtsG (split forward only): the world points live in the candidate's global
// FK record (buf.fk, read through L1 / L2) instead of shared memory, for hands
// whose 24 N bytes of points would cap the forward at one CTA per SM.
template <class Sdf, int Phase, bool PtsG = false, bool Multi = false>
__device__ __forceinline__ void kernel_body(const KHand& H, const KObj& O, const Sdf& sdf, const KSim& S,
                                            const KOpt& P, const KBuf& buf, int mode) {
  extern __shared__ __align__(16) unsigned char smem[];
  const SmemLayout lay(H.N, H.L, S.M, Phase == kPhaseFwd ? 0 : S.seg_max, !PtsG);  // the forward stages nothing
  double* px = reinterpret_cast<double*>(smem + lay.off_px);
  double* py = reinterpret_cast<double*>(smem + lay.off_py);
  double* pz = reinterpret_cast<double*>(smem + lay.off_pz);
  double* link = reinterpret_cast<double*>(smem + lay.off_link);
  double* ft_all = reinterpret_cast<double*>(smem + lay.off_ft);
  unsigned* bitmap_all = reinterpret_cast<unsigned*>(smem + lay.off_bitmap);
  double* stage_all = reinterpret_cast<double*>(smem + lay.off_stage);
  double* misc = reinterpret_cast<double*>(smem + lay.off_misc);
  double* sq = misc;               // [40] configuration
  double* sg = misc + 40;          // [3*32] d_stable, d_qrange, d_qlimit
  int* snext = reinterpret_cast<int*>(misc + 136);  // [1] next claimed candidate
  double* sres = reinterpret_cast<double*>(smem + lay.off_sres);  // [M] residuals
  int* sflag = reinterpret_cast<int*>(smem + lay.off_sflag);      // [M] per-sim status, [M] candidate status

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int M = S.M, N = H.N, L = H.L, J = H.J, D = 6 + J, Qd = 7 + J;
  const int W = static_cast<int>(blockDim.x >> 5);  // warp w runs sims w, w + W, ... (W = min(M, 7))
  const bool record = mode != kModeEval;
  const int nwords = (N + 31) / 32;

  SimEnv e;
  e.lane = lane;
  e.N = N;
  e.gs = S.gs;
  e.px = px; e.py = py; e.pz = pz;
  e.sample_link = H.sample_link;
  e.bitmap = bitmap_all + warp * nwords;

  e.stage = stage_all + warp * lay.stage_per_warp;
  e.seg_max = S.seg_max;
  e.ft = ft_all + warp * 6 * L;
  const size_t wslot = static_cast<size_t>(blockIdx.x) * W + warp;  // fused scratch: per (CTA, warp)
  // logs: per resident (CTA, warp) when fused; per (candidate, sim) when split
  // (bound per candidate below)
  e.slot_cap = buf.slot_stride;
  auto bind_logs = [&](size_t ws) {
    e.corr = buf.corr + ws * buf.cap_corr;
    e.slots = buf.slots + ws * buf.slot_stride;
    e.slot_of_point = buf.slot_of_point + ws * N;
    e.fric_order = buf.fric_order + ws * buf.slot_stride;
  };
  bind_logs(wslot);
  e.gft = buf.ft_global + wslot * 6 * L;
  e.cmat = buf.cmat + wslot * static_cast<size_t>(kCorrBatch) * kCorrMat;
  e.L = L;
  e.cap_corr = buf.cap_corr;
  e.O = &O;
  e.alpha = S.alpha;
  e.mu = S.mu;
  e.dt = S.dt;
  e.point_grads = nullptr;
  e.pts_global = PtsG ? 1 : 0;
  e.fold = S.fold;
  e.discard = S.discard;
  e.mcache = buf.mesh_cache ? buf.mesh_cache + wslot * static_cast<size_t>(S.gs) * N * S.steps : nullptr;
  e.mcert = buf.mesh_cert ? buf.mesh_cert + wslot * 4 * static_cast<size_t>(N) : nullptr;
  e.mcf = buf.mesh_cf ? buf.mesh_cf + wslot * static_cast<size_t>(kCertFaces + 1) * N : nullptr;

  const int k0 = mode == kModeOpt ? P.k_begin : 0;
  const int k1 = mode == kModeOpt ? P.k_end : 1;

  for (int b = blockIdx.x; b < buf.B; b = next_candidate(buf, b, snext)) {
    DGX_ASSERT(b >= 0);
    // a candidate that failed at an earlier iterate of this call stays there
    // (a multi-iterate launch's loop stops at its first failure)
    if (mode == kModeOpt && P.k_begin > P.traj_k0 && buf.status[b] != kOk) continue;
    // Adam state in registers of lanes < D of warp 0
    double am = 0.0, av = 0.0;
    double b1t = 1.0, b2t = 1.0;
    if (tid < Qd) sq[tid] = buf.q[static_cast<size_t>(b) * Qd + tid];
    if (mode == kModeOpt) {
      if (tid < D) {
        am = buf.adam_m[static_cast<size_t>(b) * D + tid];
        av = buf.adam_v[static_cast<size_t>(b) * D + tid];
      }
      for (int k = 0; k < P.k_begin; ++k) { b1t = b1t * P.beta1; b2t = b2t * P.beta2; }
    }
    int cand_status = kOk;
    __syncthreads();

    for (int k = k0; k < k1; ++k) {
      double radius = S.radius;
      if (mode == kModeOpt)
        radius = P.iters > 1 ? P.r0 * (1.0 - static_cast<double>(k) / static_cast<double>(P.iters - 1)) : 0.0;
      // 1. FK. Split execution: the forward kernel stores the link transforms
      // and world points per candidate; the adjoint kernel reloads them.
      double* fkb = Phase != kPhaseFused && (record || PtsG) ? buf.fk + static_cast<size_t>(b) * (12 * L + 3 * N)
                                                               : nullptr;
      if constexpr (PtsG) {
        px = fkb + 12 * L;
        py = fkb + 12 * L + N;
        pz = fkb + 12 * L + 2 * N;
        e.px = px; e.py = py; e.pz = pz;
      }
      for (int t = tid; t < 6 * L * M; t += blockDim.x) ft_all[t] = 0.0;
      for (int t = tid; t <= M; t += blockDim.x) sflag[t] = kOk;
      if constexpr (Phase == kPhaseAdj) {
        for (int t = tid; t < 12 * L; t += blockDim.x) link[t] = __ldcg(fkb + t);
        for (int i = tid; i < N; i += blockDim.x) {
          px[i] = __ldcg(fkb + 12 * L + i);
          py[i] = __ldcg(fkb + 12 * L + N + i);
          pz[i] = __ldcg(fkb + 12 * L + 2 * N + i);
        }
        __syncthreads();
      } else {
        if (warp == 0) link_transforms_warp(H, sq, record, link, lane);
        __syncthreads();
        for (int i = tid; i < N; i += blockDim.x) {
          const int li = H.sample_link[i];
          const double* Rl = link + 12 * li;
          M3 R;
          for (int m = 0; m < 9; ++m) R.m[m] = Rl[m];
          const V3 s{H.samples[3 * i], H.samples[3 * i + 1], H.samples[3 * i + 2]};
          const V3 p = mul(R, s) + V3{Rl[9], Rl[10], Rl[11]};
          px[i] = p.x; py[i] = p.y; pz[i] = p.z;  // PtsG: plain stores into buf.fk (read back via L1)
          if (fkb && !PtsG) {
            __stcg(fkb + 12 * L + i, p.x);
            __stcg(fkb + 12 * L + N + i, p.y);
            __stcg(fkb + 12 * L + 2 * N + i, p.z);
          }
        }
        if (fkb)
          for (int t = tid; t < 12 * L; t += blockDim.x) __stcg(fkb + t, link[t]);
        __syncthreads();
      }

      // 2-3. perturbation sims: warp w runs sims w, w + W, ...
      for (int m = warp; m < M; m += W) {
        if constexpr (Phase != kPhaseFused) bind_logs(static_cast<size_t>(b) * M + m);  // per (candidate, sim)
        e.ft = ft_all + m * 6 * L;
        e.radius = radius;
        e.point_grads = buf.point_grads ? buf.point_grads + (static_cast<size_t>(b) * M + m) * N * 3 : nullptr;
        SimStats st;
        int status = kOk;
        FtAcc acc;
        const double* vv = m < kMaxSims ? S.vel[m] : S.vel_dev + 3 * m;
        const V3 vm{vv[0], vv[1], vv[2]};
        const bool meas = mode == kModeEval && S.measure_residual;
        PROF_T(tsim);
        FwdRec* rec = Phase != kPhaseFused ? buf.fwd + static_cast<size_t>(b) * M + m : nullptr;
        double res;
        if constexpr (Multi)  // StabilityProtocol::steps > 1 (fused kernel only)
          res = run_sim_steps(sdf, e, vm, record, meas, st, status, acc,
                              buf.steps + wslot * static_cast<size_t>(S.steps), S.steps);
        else
          res = run_sim<Phase>(sdf, e, vm, record, meas, st, status, acc, rec);
        PROF_ACC(12, tsim);
        if constexpr (Phase == kPhaseFwd) {
          if (lane == 0) {
            rec->residual = res;
            rec->status = status;
          }
        }
        ft_flush_warp(acc, e.ft, lane);
        __syncwarp();
        if (lane == 0) {
          sres[m] = res;
          sflag[m] = status;
          if (buf.sim_res) buf.sim_res[static_cast<size_t>(b) * M + m] = res;
          if (buf.stats && mode == kModeEval) {
            double* so = buf.stats + (static_cast<size_t>(b) * M + m) * 5;
            so[0] = st.active; so[1] = st.corrections; so[2] = st.singular; so[3] = st.max_pen; so[4] = st.max_fric;
          }
        }
        if (Phase != kPhaseFwd && buf.sim_grads && record) {  // debug: per-perturbation gradient via the FK adjoint
          __syncwarp();
          double* ftw = e.stage;  // reuse the stage buffer (>= 6L + kMaxDim doubles)
          double* gw = e.stage + 6 * L;
          for (int t = lane; t < 6 * L; t += 32) ftw[t] = e.ft[t];
          __syncwarp();
          fk_adjoint(H, sq, link, ftw, gw, lane);
          double* o = buf.sim_grads + (static_cast<size_t>(b) * M + m) * D;
          for (int t = lane; t < D; t += 32) o[t] = gw[t];
          __syncwarp();
        }
      }
      __syncthreads();
      if constexpr (Phase == kPhaseFwd) {
        if (record) continue;  // losses / gradient / step: the adjoint kernel
      }

      // 4. losses, gradient, optimizer (warp 0)
      if (warp == 0) {
        candidate_epilogue(H, S, P, buf, mode, b, k, lane, sflag, sres, ft_all, link, stage_all, sg, sq, am, av, b1t,
                           b2t, cand_status);
        if (lane == 0) sflag[M] = cand_status;
      }
      __syncthreads();
      cand_status = sflag[M];
      if (cand_status != kOk) break;
    }
    if constexpr (Phase == kPhaseFwd) {
      if (record) {
        __syncthreads();
        continue;
      }
    }
    if constexpr (Phase == kPhaseAdj) {  // the forward's FK record of this candidate is consumed
      if (S.discard && record)
        l2_discard(buf.fk + static_cast<size_t>(b) * (12 * L + 3 * N), sizeof(double) * (12 * L + 3 * N), tid,
                   blockDim.x);
    }
    // write back
    if (mode == kModeOpt) {
      if (tid < Qd) buf.q[static_cast<size_t>(b) * Qd + tid] = sq[tid];
      if (tid < D) {
        buf.adam_m[static_cast<size_t>(b) * D + tid] = am;
        buf.adam_v[static_cast<size_t>(b) * D + tid] = av;
      }
    }
    if (tid == 0) buf.status[b] = cand_status;
    __syncthreads();
  }
}


// fused / adjoint instances: the register budget follows CTAs per SM
template <class Sdf, int Occ = CtasPerSm<Sdf>::value, int Phase = kPhaseFused, bool Multi = false>
__global__ void __launch_bounds__(224, Occ) fused_kernel(const __grid_constant__ KHand H, const __grid_constant__ KObj O,
                                                         const __grid_constant__ Sdf sdf, const __grid_constant__ KSim S,
                                                         const __grid_constant__ KOpt P, const __grid_constant__ KBuf buf,
                                                         int mode) {
  kernel_body<Sdf, Phase, false, Multi>(H, O, sdf, S, P, buf, mode);
}

// forward instance of split execution: kFwdCtasPerSm CTAs per SM. The
// register file is split per SM sub-partition (16384 each), so 14 warps on 4
// sub-partitions allow 4096 / 32 = 128 registers per thread; __maxnreg__(144)
// leaves one CTA per SM (90k vs 101k cand-iter/s)
template <class Sdf, bool PtsG = false>
__global__ void __launch_bounds__(224, PtsG ? kFwdCtasPerSmPtsG : kFwdCtasPerSm) fwd_kernel(const __grid_constant__ KHand H, const __grid_constant__ KObj O,
                                                                 DGX_FWD_SDF_GC Sdf sdf, const __grid_constant__ KSim S,
                                                                 const __grid_constant__ KOpt P, const __grid_constant__ KBuf buf,
                                                                 int mode) {
  kernel_body<Sdf, kPhaseFwd, PtsG>(H, O, sdf, S, P, buf, mode);
}

// ---------------------------------------------------------------------------
// Split adjoint as independent warp tasks (kPhaseAdjTask). A task is one
// (candidate, sim) pair claimed from the launch's ticket counter; the warp
// reads the forward's link transforms and world points from global memory
// (buf.fk, L2-resident), replays the sim's logs in reverse (run_sim), folds
// its link force / torque sums and writes them with its residual and status
// per (candidate, sim). The warp that completes a candidate's last sim (a
// per-candidate counter, release / acquire through __threadfence) runs the
// candidate's epilogue (candidate_epilogue: loss reductions in sim order, FK
// adjoint, Adam, step) from __ldcg copies of those rows. No warp waits for
// another, so sims of uneven cost do not idle the SM at a barrier, and the
// CTA size is not tied to M.
template <class Sdf>
__device__ __forceinline__ void adj_task_body(const KHand& H, const KObj& O, const Sdf& sdf, const KSim& S,
                                              const KOpt& P, const KBuf& buf, int mode) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int M = S.M, N = H.N, L = H.L, J = H.J, D = 6 + J, Qd = 7 + J;
  const TaskLayout lay(L, M, S.seg_max);
  double* wb = reinterpret_cast<double*>(smem) + static_cast<size_t>(warp) * lay.per_warp;
  double* stage = wb;
  double* ftw = wb + lay.off_ft;
  double* sq = wb + lay.off_sq;
  double* sg = wb + lay.off_sg;
  const int gwarp = static_cast<int>(blockIdx.x) * kTaskWarps + warp;
  // CTA task queue (after the warps' areas): the CTA's warps take the sims of
  // the same few candidates, so those candidates' points stay in the SM's L1
  unsigned char* qbase = smem + 8 * static_cast<size_t>(lay.per_warp) * kTaskWarps;
  int* q_next = reinterpret_cast<int*>(qbase);
  unsigned long long* q_ring = reinterpret_cast<unsigned long long*>(qbase + 16);
  int* q_done = reinterpret_cast<int*>(qbase + 16 + 8 * kTaskRing);
  if (threadIdx.x == 0) *q_next = 0;
  if (threadIdx.x < kTaskRing) {
    q_ring[threadIdx.x] = 0ull;
    q_done[threadIdx.x] = M;  // slot never used: free
  }
  __syncthreads();

  SimEnv e;
  e.lane = lane;
  e.N = N;
  e.gs = S.gs;
  e.sample_link = H.sample_link;
  e.bitmap = nullptr;
  e.stage = stage;
  e.seg_max = S.seg_max;
  e.ft = ftw;
  e.gft = buf.ft_global + static_cast<size_t>(gwarp) * 6 * L;
  e.cmat = buf.cmat + static_cast<size_t>(gwarp) * kCorrBatch * kCorrMat;
  e.L = L;
  e.cap_corr = buf.cap_corr;
  e.slot_cap = buf.slot_stride;
  e.O = &O;
  e.alpha = S.alpha;
  e.mu = S.mu;
  e.dt = S.dt;
  e.mcache = nullptr;
  e.mcert = nullptr;
  e.mcf = nullptr;
  e.pts_global = 1;
  e.fold = S.fold;
  e.discard = S.discard;
  const int k = mode == kModeOpt ? P.k_begin : 0;
  e.radius = S.radius;
  if (mode == kModeOpt)
    e.radius = P.iters > 1 ? P.r0 * (1.0 - static_cast<double>(k) / static_cast<double>(P.iters - 1)) : 0.0;
  // next task of this warp: task j of the CTA is sim j % M of its candidate
  // slot j / M. The warp that takes sim 0 claims the slot's candidate (the
  // CTA's first slot: blockIdx.x; later ones: a launch ticket + gridDim.x) and
  // publishes it tagged with the slot; the other sims' warps read it. A ring
  // entry is reused only after all M sims of its previous slot read it.
  auto next_task = [&](int& b, int& m) {
    int cb = 0, cm = 0;
    if (lane == 0) {
      const int j = atomicAdd(q_next, 1);
      const int c = j / M;
      cm = j - c * M;
      const int r = c % kTaskRing;
      volatile unsigned long long* ring = q_ring;
      volatile int* done = q_done;
      if (cm == 0) {
        while (done[r] < M) {
        }
        int cand = static_cast<int>(blockIdx.x) + c * static_cast<int>(gridDim.x);  // static (no counter)
        if (c > 0 && buf.claim)
          cand = static_cast<int>(min(atomicAdd(buf.claim, 1ull), static_cast<unsigned long long>(INT_MAX / 2))) +
                 static_cast<int>(gridDim.x);
        done[r] = 0;
        __threadfence_block();
        ring[r] = (static_cast<unsigned long long>(c + 1) << 32) | static_cast<unsigned int>(cand);
      }
      unsigned long long v;
      do {
        v = ring[r];
      } while (static_cast<int>(v >> 32) != c + 1);
      cb = static_cast<int>(v & 0xffffffffull);
      atomicAdd(q_done + r, 1);
    }
    b = __shfl_sync(kFull, cb, 0);
    m = __shfl_sync(kFull, cm, 0);
  };
  int b = 0, m = 0;
  next_task(b, m);
  while (b < buf.B) {
    const size_t bm = static_cast<size_t>(b) * M + m;
    const bool skip = mode == kModeOpt && P.k_begin > P.traj_k0 && buf.status[b] != kOk;
    if (!skip) {
      e.corr = buf.corr + bm * buf.cap_corr;
      e.slots = buf.slots + bm * buf.slot_stride;
      e.slot_of_point = buf.slot_of_point + bm * N;
      e.fric_order = buf.fric_order + bm * buf.slot_stride;
      const double* fkb = buf.fk + static_cast<size_t>(b) * (12 * L + 3 * N);
      e.px = fkb + 12 * L;
      e.py = fkb + 12 * L + N;
      e.pz = fkb + 12 * L + 2 * N;
      e.point_grads = buf.point_grads ? buf.point_grads + bm * N * 3 : nullptr;
      for (int i = lane; i < 6 * L; i += 32) ftw[i] = 0.0;
      __syncwarp();
      SimStats st;
      int status = kOk;
      FtAcc acc;
      const double* vv = m < kMaxSims ? S.vel[m] : S.vel_dev + 3 * m;
      const V3 vm{vv[0], vv[1], vv[2]};
      const double res = run_sim<kPhaseAdjTask>(sdf, e, vm, true, false, st, status, acc, buf.fwd + bm);
      ft_flush_warp(acc, ftw, lane);
      __syncwarp();
      for (int i = lane; i < 6 * L; i += 32) __stcg(buf.task_ft + bm * 6 * L + i, ftw[i]);
      if (lane == 0) {
        __stcg(buf.task_res + bm, res);
        __stcg(buf.task_stat + bm, status);
        if (buf.sim_res) buf.sim_res[bm] = res;
      }
      if (buf.sim_grads) {  // debug: per-perturbation gradient via the FK adjoint
        if (lane < Qd) sq[lane] = buf.q[static_cast<size_t>(b) * Qd + lane];
        double* ftc = stage;
        for (int i = lane; i < 6 * L; i += 32) ftc[i] = ftw[i];
        __syncwarp();
        fk_adjoint(H, sq, fkb, ftc, sg, lane);
        for (int i = lane; i < D; i += 32) buf.sim_grads[bm * D + i] = sg[i];
        __syncwarp();
      }
    }
    // publish this sim, then count it; the candidate's last sim runs its epilogue
    __threadfence();
    __syncwarp();
    int prev = 0;
    if (lane == 0) prev = atomicAdd(buf.task_done + b, 1);
    prev = __shfl_sync(kFull, prev, 0);
    if (prev == M - 1 && !skip) {
      __threadfence();  // acquire: the other sims' rows are visible
      const size_t b0 = static_cast<size_t>(b) * M;
      double* ft_all = stage;                        // [M][6L]
      double* sres = stage + M * 6 * L;              // [M]
      int* sflag = reinterpret_cast<int*>(sres + M); // [M]
      double* scratch = sres + M + (M + 1) / 2 + 1;  // [6L]
      for (int i = lane; i < M * 6 * L; i += 32) ft_all[i] = __ldcg(buf.task_ft + b0 * 6 * L + i);
      for (int i = lane; i < M; i += 32) {
        sres[i] = __ldcg(buf.task_res + b0 + i);
        sflag[i] = __ldcg(buf.task_stat + b0 + i);
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
      int cand_status = kOk;
      const double* link = buf.fk + static_cast<size_t>(b) * (12 * L + 3 * N);
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
      if (S.discard) {  // every sim of the candidate has read its FK record; the task rows are consumed
        l2_discard(link, sizeof(double) * (12 * L + 3 * N), lane, 32);
        l2_discard(buf.task_ft + b0 * 6 * L, sizeof(double) * M * 6 * L, lane, 32);
      }
    }
    next_task(b, m);
  }
}

template <class Sdf, int MinBlocks>
__global__ void __launch_bounds__(32 * kTaskWarps, MinBlocks) adj_task_kernel(const __grid_constant__ KHand H, const __grid_constant__ KObj O,
                                                                              const __grid_constant__ Sdf sdf, const __grid_constant__ KSim S,
                                                                              const __grid_constant__ KOpt P, const __grid_constant__ KBuf buf,
                                                                              int mode) {
  adj_task_body<Sdf>(H, O, sdf, S, P, buf, mode);
}

#include "dgx_lane_adj.cuh"
}  // namespace dgx

// ---------------------------------------------------------------------------
// FK-only and apply_gradient_step kernels (HandModel::forward, hand.hpp:86;
// apply_gradient_step, losses.cpp:92-102)
// ---------------------------------------------------------------------------
namespace dgx {

__global__ void __launch_bounds__(256) forward_kernel(KHand H, const double* q, double* out, int B) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* link = reinterpret_cast<double*>(smem);
  double* sq = link + 12 * H.L;
  const int Qd = 7 + H.J;
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    if (threadIdx.x < Qd) sq[threadIdx.x] = q[static_cast<size_t>(b) * Qd + threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0) link_transforms(H, sq, false, link);
    __syncthreads();
    for (int i = threadIdx.x; i < H.N; i += blockDim.x) {
      const double* Rl = link + 12 * H.sample_link[i];
      M3 R;
      for (int m = 0; m < 9; ++m) R.m[m] = Rl[m];
      const V3 p = mul(R, V3{H.samples[3 * i], H.samples[3 * i + 1], H.samples[3 * i + 2]}) + V3{Rl[9], Rl[10], Rl[11]};
      double* o = out + (static_cast<size_t>(b) * H.N + i) * 3;
      o[0] = p.x; o[1] = p.y; o[2] = p.z;
    }
    __syncthreads();
  }
}

// Contact generation (the reference specifies but does not
// implement it): per candidate, FK (hand.hpp:116-152), every hand sample
// queried against the object at its canonical pose (object frame = world),
// contact when |rho| <= threshold. Per threshold: contact count and contact
// area (sum of HandModel::sample_areas over contacts) from fixed-
// order reductions; the contacts at the largest threshold are compacted in
// point order (ballot prefix sums) with (rho, smoothed point, unit gradient).
constexpr int kMaxThresholds = 16;

template <class Sdf>
__global__ void __launch_bounds__(256) contacts_kernel(const __grid_constant__ KHand H, const __grid_constant__ Sdf sdf, int B, const double* __restrict__ q,
                                                       const double* __restrict__ area, int T,
                                                       const double* __restrict__ thr, int cap,
                                                       double* __restrict__ ca, int* __restrict__ cnt,
                                                       int* __restrict__ ncont, int* __restrict__ cidx,
                                                       double* __restrict__ crec) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* link = reinterpret_cast<double*>(smem);
  double* sq = link + 12 * H.L;
  double* red = sq + 48;                                  // [8 warps][T]
  int* redc = reinterpret_cast<int*>(red + 8 * kMaxThresholds);  // [8 warps][T]
  int* wtot = redc + 8 * kMaxThresholds;                  // [8]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  const int Qd = 7 + H.J, N = H.N;
  const double tmax = thr[T - 1];
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    if (tid < Qd) sq[tid] = q[static_cast<size_t>(b) * Qd + tid];
    __syncthreads();
    if (tid == 0) link_transforms(H, sq, false, link);
    __syncthreads();
    double acc[kMaxThresholds];
    int ac[kMaxThresholds];
#pragma unroll
    for (int t = 0; t < kMaxThresholds; ++t) { acc[t] = 0.0; ac[t] = 0; }
    int nbase = 0;
    for (int c = 0; c < N; c += blockDim.x) {
      const int i = c + tid;
      bool con = false;
      SdfQuery qq{};
      if (i < N) {
        const double* Rl = link + 12 * H.sample_link[i];
        M3 R;
        for (int m = 0; m < 9; ++m) R.m[m] = Rl[m];
        const V3 p = mul(R, V3{H.samples[3 * i], H.samples[3 * i + 1], H.samples[3 * i + 2]}) + V3{Rl[9], Rl[10], Rl[11]};
        qq = sdf.query(p);
        const double ar = fabs(qq.rho);
        const double ai = area[i];
#pragma unroll
        for (int t = 0; t < kMaxThresholds; ++t)
          if (t < T && ar <= thr[t]) { acc[t] += ai; ++ac[t]; }
        con = ar <= tmax;
      }
      const unsigned m = __ballot_sync(0xffffffffu, con);
      if (lane == 0) wtot[warp] = __popc(m);
      __syncthreads();
      int off = nbase, tot = 0;
      for (int w = 0; w < nwarp; ++w) {
        if (w < warp) off += wtot[w];
        tot += wtot[w];
      }
      off += __popc(m & ((1u << lane) - 1u));
      if (con && off < cap) {
        const size_t k = static_cast<size_t>(b) * cap + off;
        cidx[k] = i;
        double* r = crec + 7 * k;
        r[0] = qq.rho;
        r[1] = qq.proxy.x; r[2] = qq.proxy.y; r[3] = qq.proxy.z;
        r[4] = qq.grad.x; r[5] = qq.grad.y; r[6] = qq.grad.z;
      }
      nbase += tot;
      __syncthreads();
    }
    // fixed-order reductions: xor butterfly per warp, then warps in order
#pragma unroll
    for (int t = 0; t < kMaxThresholds; ++t) {
      if (t >= T) break;
      double v = acc[t];
      int n = ac[t];
      for (int o = 16; o > 0; o >>= 1) {
        v += __shfl_xor_sync(0xffffffffu, v, o);
        n += __shfl_xor_sync(0xffffffffu, n, o);
      }
      if (lane == 0) {
        red[warp * kMaxThresholds + t] = v;
        redc[warp * kMaxThresholds + t] = n;
      }
    }
    __syncthreads();
    if (tid < T) {
      double v = 0.0;
      int n = 0;
      for (int w = 0; w < nwarp; ++w) {
        v += red[w * kMaxThresholds + tid];
        n += redc[w * kMaxThresholds + tid];
      }
      ca[static_cast<size_t>(b) * T + tid] = v;
      cnt[static_cast<size_t>(b) * T + tid] = n;
    }
    if (tid == 0) ncont[b] = nbase;
    __syncthreads();
  }
}

// Grasp-energy terms (north_star (3); no reference counterpart, so
// parity-unpinned; dgx.h dgx_grasp_energy_batch): one CTA (8 warps) per
// candidate. FK (hand.hpp:116-152), every hand sample queried at the object's
// canonical pose (object frame = world, as the contact generation above);
// contacts C = {|rho| <= thr}. E_fc = |sum_C n|^2 + |sum_C (p - com) x n|^2 / l^2,
// E_pen = sum max(0, -rho). Gradients with the contact set and normals frozen
// (sim.hpp:102-104 convention): dE_fc/dp = 2 (n x tau) / l^2 on C, dE_pen/dp =
// -n where rho < 0, folded per link into force / torque sums (segmented warp
// scans over the point-ordered samples, then warps in order: deterministic)
// and mapped to [pos | tangent | joints] by fk_adjoint. Outputs: e [B,2],
// g [B,2,D] and / or gw [B,D] = w_fc dE_fc + w_pen dE_pen (optimizer).
constexpr int kEnergyWarps = 8;

__device__ __forceinline__ void seg_flush12(double (&v)[12], int key, double* ftw, int lane) {
  // inclusive segmented scan over equal consecutive keys (samples are in link
  // order, so each link is one lane range); the segment's last lane adds it
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int kk = __shfl_up_sync(kFull, key, d);
    double u[12];
#pragma unroll
    for (int c = 0; c < 12; ++c) u[c] = __shfl_up_sync(kFull, v[c], d);
    if (lane >= d && kk == key) {
#pragma unroll
      for (int c = 0; c < 12; ++c) v[c] += u[c];
    }
  }
  const int knext = __shfl_down_sync(kFull, key, 1);
  if (key >= 0 && (lane == 31 || knext != key)) {
    double* f = ftw + 12 * key;
#pragma unroll
    for (int c = 0; c < 12; ++c) f[c] += v[c];
  }
  __syncwarp();
}

template <class Sdf>
__global__ void __launch_bounds__(32 * kEnergyWarps) energy_kernel(const __grid_constant__ KHand H, const __grid_constant__ KObj O,
                                                                  const __grid_constant__ Sdf sdf, const __grid_constant__ KSim S, int B, const double* __restrict__ q,
                                                                  const int* __restrict__ status,
                                                                  double* __restrict__ e_out,
                                                                  double* __restrict__ g_out,
                                                                  double* __restrict__ gw_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L = H.L, N = H.N, D = 6 + H.J, Qd = 7 + H.J;
  double* link = reinterpret_cast<double*>(smem);                 // [12 L]
  double* sq = link + 12 * L;                                     // [40]
  double* red = sq + 40;                                          // [8 warps][8]
  double* ftw = red + 8 * kEnergyWarps;                           // [8 warps][L][12]
  double* ftf = ftw + kEnergyWarps * 12 * L;                      // [6 L] force closure
  double* ftp = ftf + 6 * L;                                      // [6 L] penetration
  double* gg = ftp + 6 * L;                                       // [2][32]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double inv_l2 = 1.0 / (S.fc_scale * S.fc_scale);
  for (int b = blockIdx.x; b < B; b += gridDim.x) {
    if (status && status[b] != kOk) continue;  // failed earlier in this optimizer call
    if (tid < Qd) sq[tid] = q[static_cast<size_t>(b) * Qd + tid];
    for (int t = tid; t < kEnergyWarps * 12 * L; t += blockDim.x) ftw[t] = 0.0;
    __syncthreads();
    if (warp == 0) link_transforms_warp(H, sq, false, link, lane);
    __syncthreads();
    // pass 1: contact sums f, tau and the penetration sum (fixed-order reduction)
    double acc[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int i = tid; i < N; i += blockDim.x) {
      const double* Rl = link + 12 * H.sample_link[i];
      M3 R;
      for (int m = 0; m < 9; ++m) R.m[m] = Rl[m];
      const V3 p = mul(R, V3{H.samples[3 * i], H.samples[3 * i + 1], H.samples[3 * i + 2]}) + V3{Rl[9], Rl[10], Rl[11]};
      const SdfQuery qq = sdf.query(p);
      if (fabs(qq.rho) <= S.fc_thr) {
        const V3 tq = cross(p - O.com, qq.grad);
        acc[0] += qq.grad.x; acc[1] += qq.grad.y; acc[2] += qq.grad.z;
        acc[3] += tq.x; acc[4] += tq.y; acc[5] += tq.z;
      }
      if (qq.rho < 0.0) acc[6] -= qq.rho;
    }
#pragma unroll
    for (int c = 0; c < 7; ++c) acc[c] = warp_sum(acc[c]);
    if (lane == 0)
      for (int c = 0; c < 7; ++c) red[8 * warp + c] = acc[c];
    __syncthreads();
    double tot[7];
#pragma unroll
    for (int c = 0; c < 7; ++c) {
      tot[c] = 0.0;
      for (int w = 0; w < kEnergyWarps; ++w) tot[c] += red[8 * w + c];
    }
    const V3 f{tot[0], tot[1], tot[2]}, tau{tot[3], tot[4], tot[5]};
    const double e_fc = dot(f, f) + dot(tau, tau) * inv_l2, e_pen = tot[6];
    // pass 2: per-sample gradients folded into per-link force / torque sums
    // (12 per link: force closure F, T | penetration F, T); chunks of 32
    // consecutive samples, chunk c on warp c % 8
    for (int c0 = 32 * warp; c0 < N; c0 += 32 * kEnergyWarps) {
      const int i = c0 + lane;
      double v[12];
#pragma unroll
      for (int c = 0; c < 12; ++c) v[c] = 0.0;
      int key = -1;
      if (i < N) {
        key = H.sample_link[i];
        const double* Rl = link + 12 * key;
        M3 R;
        for (int m = 0; m < 9; ++m) R.m[m] = Rl[m];
        const V3 p = mul(R, V3{H.samples[3 * i], H.samples[3 * i + 1], H.samples[3 * i + 2]}) + V3{Rl[9], Rl[10], Rl[11]};
        const SdfQuery qq = sdf.query(p);
        if (fabs(qq.rho) <= S.fc_thr) {
          const V3 gp = cross(qq.grad, tau) * (2.0 * inv_l2);
          const V3 tq = cross(p, gp);
          v[0] = gp.x; v[1] = gp.y; v[2] = gp.z; v[3] = tq.x; v[4] = tq.y; v[5] = tq.z;
        }
        if (qq.rho < 0.0) {
          const V3 gp = qq.grad * -1.0;
          const V3 tq = cross(p, gp);
          v[6] = gp.x; v[7] = gp.y; v[8] = gp.z; v[9] = tq.x; v[10] = tq.y; v[11] = tq.z;
        }
      }
      seg_flush12(v, key, ftw + warp * 12 * L, lane);
    }
    __syncthreads();
    for (int t = tid; t < 6 * L; t += blockDim.x) {
      const int l = t / 6, c = t - 6 * l;
      double sf = 0.0, sp = 0.0;
      for (int w = 0; w < kEnergyWarps; ++w) {
        sf += ftw[(w * L + l) * 12 + c];
        sp += ftw[(w * L + l) * 12 + 6 + c];
      }
      ftf[t] = sf;
      ftp[t] = sp;
    }
    __syncthreads();
    if (warp == 0) fk_adjoint(H, sq, link, ftf, gg, lane);
    if (warp == 1) fk_adjoint(H, sq, link, ftp, gg + 32, lane);
    __syncthreads();
    if (tid < D) {
      const double gf = gg[tid], gp = gg[32 + tid];
      if (g_out) {
        g_out[static_cast<size_t>(b) * 2 * D + tid] = gf;
        g_out[static_cast<size_t>(b) * 2 * D + D + tid] = gp;
      }
      if (gw_out) gw_out[static_cast<size_t>(b) * D + tid] = S.w_fc * gf + S.w_pen * gp;
    }
    if (tid == 0 && e_out) {
      e_out[2 * static_cast<size_t>(b)] = e_fc;
      e_out[2 * static_cast<size_t>(b) + 1] = e_pen;
    }
    __syncthreads();
  }
}

cudaError_t launch_energy(const KHand& H, const KObj& O, const SdfSet& sdf, const KSim& S, int B, const double* q,
                          const int* status, double* e, double* g, double* gw, int grid, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  const size_t smem = sizeof(double) * (12 * H.L + 40 + 8 * kEnergyWarps + kEnergyWarps * 12 * H.L + 12 * H.L + 64);
  const int th = 32 * kEnergyWarps;
  switch (sdf.kind) {
    case kSdfSphere: energy_kernel<<<grid, th, smem, st>>>(H, O, sdf.sph, S, B, q, status, e, g, gw); break;
    case kSdfBox: energy_kernel<<<grid, th, smem, st>>>(H, O, sdf.box, S, B, q, status, e, g, gw); break;
    case kSdfGrid: energy_kernel<<<grid, th, smem, st>>>(H, O, sdf.grd, S, B, q, status, e, g, gw); break;
    case kSdfMesh: energy_kernel<<<grid, th, smem, st>>>(H, O, sdf.mesh, S, B, q, status, e, g, gw); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_contacts(const KHand& H, const SdfSet& sdf, int B, const double* q, const double* area, int T,
                            const double* thr, int cap, double* ca, int* cnt, int* ncont, int* cidx, double* crec,
                            int grid, cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  const size_t smem = sizeof(double) * (12 * H.L + 48 + 8 * kMaxThresholds) + sizeof(int) * (8 * kMaxThresholds + 8);
  switch (sdf.kind) {
    case kSdfSphere:
      contacts_kernel<<<grid, 256, smem, st>>>(H, sdf.sph, B, q, area, T, thr, cap, ca, cnt, ncont, cidx, crec);
      break;
    case kSdfBox:
      contacts_kernel<<<grid, 256, smem, st>>>(H, sdf.box, B, q, area, T, thr, cap, ca, cnt, ncont, cidx, crec);
      break;
    case kSdfGrid:
      contacts_kernel<<<grid, 256, smem, st>>>(H, sdf.grd, B, q, area, T, thr, cap, ca, cnt, ncont, cidx, crec);
      break;
    case kSdfMesh:
      contacts_kernel<<<grid, 256, smem, st>>>(H, sdf.mesh, B, q, area, T, thr, cap, ca, cnt, ncont, cidx, crec);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

__global__ void step_kernel(int J, const double* q, const double* g, double lr, double* out, int B) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int Qd = 7 + J, D = 6 + J;
  const double* qi = q + static_cast<size_t>(b) * Qd;
  const double* gi = g + static_cast<size_t>(b) * D;
  double* o = out + static_cast<size_t>(b) * Qd;
  o[0] = qi[0] - lr * gi[0];
  o[1] = qi[1] - lr * gi[1];
  o[2] = qi[2] - lr * gi[2];
  const V3 tangent{-lr * gi[3], -lr * gi[4], -lr * gi[5]};
  const Q4 qn = qnormalized(qmul(quat_exp(tangent), Q4{qi[3], qi[4], qi[5], qi[6]}));
  o[3] = qn.w; o[4] = qn.x; o[5] = qn.y; o[6] = qn.z;
  for (int j = 0; j < J; ++j) o[7 + j] = qi[7 + j] - lr * gi[6 + j];
}

template <class Sdf, int Occ, int Phase>
static cudaError_t allow_smem() {
  static bool configured = false;
  if (configured) return cudaSuccess;
  cudaError_t e =
      cudaFuncSetAttribute(fused_kernel<Sdf, Occ, Phase>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e == cudaSuccess) configured = true;
  return e;
}

template <class Sdf, bool PtsG>
static cudaError_t allow_smem_fwd() {
  static bool configured = false;
  if (configured) return cudaSuccess;
  cudaError_t e =
      cudaFuncSetAttribute(fwd_kernel<Sdf, PtsG>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e == cudaSuccess) configured = true;
  return e;
}

// the split pair exists for the analytic and grid backends; mesh objects run
// fused (their forward and adjoint share the per-point-sweep face cache)
template <class Sdf>
constexpr bool kSplitCapable = !std::is_same<Sdf, MeshSdf>::value;

template <class Sdf>
static cudaError_t launch_fused_t(const KHand& H, const KObj& O, const Sdf& sdf, const KSim& S, const KOpt& P,
                                  const KBuf& buf, int mode, int phase, int grid, int smem, cudaStream_t st) {
  constexpr int occ = CtasPerSm<Sdf>::value;
  cudaError_t e = cudaSuccess;
  if constexpr (kSplitCapable<Sdf>) {
    if (phase == kPhaseFwd) {
      if (S.pts_global) {
        if ((e = allow_smem_fwd<Sdf, true>()) != cudaSuccess) return e;
        fwd_kernel<Sdf, true><<<grid, 32 * S.warps(), smem, st>>>(H, O, sdf, S, P, buf, mode);
      } else {
        if ((e = allow_smem_fwd<Sdf, false>()) != cudaSuccess) return e;
        fwd_kernel<Sdf, false><<<grid, 32 * S.warps(), smem, st>>>(H, O, sdf, S, P, buf, mode);
      }
      return cudaGetLastError();
    }
    if (phase == kPhaseAdj) {
      if ((e = allow_smem<Sdf, occ, kPhaseAdj>()) != cudaSuccess) return e;
      fused_kernel<Sdf, occ, kPhaseAdj><<<grid, 32 * S.warps(), smem, st>>>(H, O, sdf, S, P, buf, mode);
      return cudaGetLastError();
    }
  }
  if (phase != kPhaseFused) return cudaErrorInvalidValue;
  if (S.steps > 1) {  // multi-step protocol instance
    static bool configured = false;
    if (!configured) {
      if ((e = cudaFuncSetAttribute(fused_kernel<Sdf, occ, kPhaseFused, true>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)) != cudaSuccess)
        return e;
      configured = true;
    }
    fused_kernel<Sdf, occ, kPhaseFused, true><<<grid, 32 * S.warps(), smem, st>>>(H, O, sdf, S, P, buf, mode);
    return cudaGetLastError();
  }
  if ((e = allow_smem<Sdf, occ, kPhaseFused>()) != cudaSuccess) return e;
  fused_kernel<Sdf, occ, kPhaseFused><<<grid, 32 * S.warps(), smem, st>>>(H, O, sdf, S, P, buf, mode);
  return cudaGetLastError();
}

// warp-task adjoint instances: kTaskMinBlocks CTAs of kTaskWarps warps per SM
// sets the register budget (2 -> 8 warps/SM at <= 255 registers; 3 -> 12
// warps at <= 168)
#ifndef DGX_TASK_MINBLOCKS
#define DGX_TASK_MINBLOCKS 1
#endif
constexpr int kTaskMinBlocks = DGX_TASK_MINBLOCKS;

template <class Sdf>
static cudaError_t task_attr() {
  static bool configured = false;
  if (configured) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(adj_task_kernel<Sdf, kTaskMinBlocks>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e == cudaSuccess) configured = true;
  return e;
}

template <class Sdf>
static cudaError_t launch_task_t(const KHand& H, const KObj& O, const Sdf& sdf, const KSim& S, const KOpt& P,
                                 const KBuf& buf, int mode, int grid, int smem, cudaStream_t st) {
  if constexpr (kSplitCapable<Sdf>) {
    cudaError_t e = task_attr<Sdf>();
    if (e != cudaSuccess) return e;
    adj_task_kernel<Sdf, kTaskMinBlocks><<<grid, 32 * kTaskWarps, smem, st>>>(H, O, sdf, S, P, buf, mode);
    return cudaGetLastError();
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_adj_task(const KHand& H, const KObj& O, const SdfSet& sdf, const KSim& S, const KOpt& P,
                            const KBuf& buf, int mode, int grid, int smem, cudaStream_t st) {
  switch (sdf.kind) {
    case kSdfSphere: return launch_task_t(H, O, sdf.sph, S, P, buf, mode, grid, smem, st);
    case kSdfBox: return launch_task_t(H, O, sdf.box, S, P, buf, mode, grid, smem, st);
    case kSdfGrid: return launch_task_t(H, O, sdf.grd, S, P, buf, mode, grid, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

template <class Sdf>
static cudaError_t task_occ_t(int smem, int* per_sm) {
  if constexpr (kSplitCapable<Sdf>) {
    cudaError_t e = task_attr<Sdf>();
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, adj_task_kernel<Sdf, kTaskMinBlocks>,
                                                         32 * kTaskWarps, smem);
  }
  return cudaErrorInvalidValue;
}

cudaError_t adj_task_occupancy(int kind, int smem, int* per_sm) {
  switch (kind) {
    case kSdfSphere: return task_occ_t<SphereSdf>(smem, per_sm);
    case kSdfBox: return task_occ_t<BoxSdf>(smem, per_sm);
    case kSdfGrid: return task_occ_t<GridSdf>(smem, per_sm);
    default: return cudaErrorInvalidValue;
  }
}

// lane adjoint (dgx_lane_adj.cuh): one thread per (candidate, sim), then one
// warp per candidate for the epilogue
template <class Sdf>
static cudaError_t launch_lane_t(const KHand& H, const KObj& O, const Sdf& sdf, const KSim& S, const KOpt& P,
                                 const KBuf& buf, int mode, cudaStream_t st) {
  if constexpr (kSplitCapable<Sdf>) {
    const long long nt = static_cast<long long>(buf.B) * S.M;
    const int grid = static_cast<int>((nt + kLaneAdjThreads - 1) / kLaneAdjThreads);
    static bool configured = false;  // small M: up to 32 candidates' staged points per warp (> 48 KB)
    if (!configured) {
      const cudaError_t e =
          cudaFuncSetAttribute(lane_adj_kernel<Sdf>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      if (e != cudaSuccess) return e;
      configured = true;
    }
    lane_adj_kernel<Sdf><<<grid, kLaneAdjThreads, lane_smem_bytes(S.M), st>>>(H, O, sdf, S, P, buf, mode);
    return cudaGetLastError();
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_lane_adj(const KHand& H, const KObj& O, const SdfSet& sdf, const KSim& S, const KOpt& P,
                            const KBuf& buf, int mode, cudaStream_t st) {
  switch (sdf.kind) {
    case kSdfSphere: return launch_lane_t(H, O, sdf.sph, S, P, buf, mode, st);
    case kSdfBox: return launch_lane_t(H, O, sdf.box, S, P, buf, mode, st);
    case kSdfGrid: return launch_lane_t(H, O, sdf.grd, S, P, buf, mode, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_lane_epi(const KHand& H, const KSim& S, const KOpt& P, const KBuf& buf, int mode, cudaStream_t st) {
  static bool configured = false;
  // kEpiWarps candidates per CTA, fewer when many sims' link sums would not fit
  const int per_warp = 8 * lane_epi_doubles(S.M, H.L);
  const int warps = std::max(1, std::min(kEpiWarps, (227 * 1024) / per_warp));
  const int smem = warps * per_warp;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(lane_epi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  lane_epi_kernel<<<(buf.B + warps - 1) / warps, 32 * warps, smem, st>>>(H, S, P, buf, mode);
  return cudaGetLastError();
}

cudaError_t launch_fused(const KHand& H, const KObj& O, const SdfSet& sdf, const KSim& S, const KOpt& P,
                         const KBuf& buf, int mode, int phase, int grid, int smem, cudaStream_t st) {
  switch (sdf.kind) {
    case kSdfSphere: return launch_fused_t(H, O, sdf.sph, S, P, buf, mode, phase, grid, smem, st);
    case kSdfBox: return launch_fused_t(H, O, sdf.box, S, P, buf, mode, phase, grid, smem, st);
    case kSdfGrid: return launch_fused_t(H, O, sdf.grd, S, P, buf, mode, phase, grid, smem, st);
    case kSdfMesh: return launch_fused_t(H, O, sdf.mesh, S, P, buf, mode, phase, grid, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

template <class Sdf, int Occ, int Phase>
static cudaError_t occupancy_i(int M, int smem, int* blocks_per_sm) {
  cudaError_t e = allow_smem<Sdf, Occ, Phase>();
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, fused_kernel<Sdf, Occ, Phase>,
                                                       32 * (M < kMaxWarps ? M : kMaxWarps), smem);
}

template <class Sdf>
static cudaError_t occupancy_t(int M, int smem, int phase, int* blocks_per_sm) {
  constexpr int occ = CtasPerSm<Sdf>::value;
  if constexpr (kSplitCapable<Sdf>) {
    if (phase == kPhaseFwd || phase == kPhaseFwdPtsG) {
      const bool g = phase == kPhaseFwdPtsG;
      cudaError_t e = g ? allow_smem_fwd<Sdf, true>() : allow_smem_fwd<Sdf, false>();
      if (e != cudaSuccess) return e;
      return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, g ? fwd_kernel<Sdf, true> : fwd_kernel<Sdf, false>,
                                                           32 * (M < kMaxWarps ? M : kMaxWarps), smem);
    }
    if (phase == kPhaseAdj) return occupancy_i<Sdf, occ, kPhaseAdj>(M, smem, blocks_per_sm);
  }
  if (phase != kPhaseFused) return cudaErrorInvalidValue;
  return occupancy_i<Sdf, occ, kPhaseFused>(M, smem, blocks_per_sm);
}

cudaError_t fused_occupancy(int kind, int M, int smem, int phase, int* blocks_per_sm) {
  switch (kind) {
    case kSdfSphere: return occupancy_t<SphereSdf>(M, smem, phase, blocks_per_sm);
    case kSdfBox: return occupancy_t<BoxSdf>(M, smem, phase, blocks_per_sm);
    case kSdfGrid: return occupancy_t<GridSdf>(M, smem, phase, blocks_per_sm);
    case kSdfMesh: return occupancy_t<MeshSdf>(M, smem, phase, blocks_per_sm);
    default: return cudaErrorInvalidValue;
  }
}

// one thread per point: MeshSdf::dilated / dilated_within (sdf.cpp:62-81) for
// any backend
template <class Sdf>
__global__ void sdf_query_kernel(Sdf sdf, int n, const double* r, double radius, int within, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const V3 p{r[3 * i], r[3 * i + 1], r[3 * i + 2]};
  double* o = out + 8 * static_cast<size_t>(i);
  if (within && sdf_culled(sdf, p, radius)) {
    o[0] = kInf;
    for (int k = 1; k < 8; ++k) o[k] = 0.0;
    return;
  }
  const SdfQuery q = sdf.query(p);
  o[0] = q.rho - radius;
  o[1] = q.grad.x; o[2] = q.grad.y; o[3] = q.grad.z;
  o[4] = q.proxy.x; o[5] = q.proxy.y; o[6] = q.proxy.z;
  o[7] = static_cast<double>(q.sign);
}

cudaError_t launch_sdf_query(const SdfSet& sdf, int n, const double* r, double radius, int within, double* out,
                             cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int blocks = (n + 127) / 128;
  switch (sdf.kind) {
    case kSdfSphere: sdf_query_kernel<<<blocks, 128, 0, st>>>(sdf.sph, n, r, radius, within, out); break;
    case kSdfBox: sdf_query_kernel<<<blocks, 128, 0, st>>>(sdf.box, n, r, radius, within, out); break;
    case kSdfGrid: sdf_query_kernel<<<blocks, 128, 0, st>>>(sdf.grd, n, r, radius, within, out); break;
    case kSdfMesh: sdf_query_kernel<<<blocks, 128, 0, st>>>(sdf.mesh, n, r, radius, within, out); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_forward(const KHand& H, const double* q, double* out, int B, int grid, cudaStream_t st) {
  const int smem = 8 * (12 * H.L + 7 + H.J + 8);
  forward_kernel<<<grid, 256, smem, st>>>(H, q, out, B);
  return cudaGetLastError();
}

cudaError_t launch_step(int J, const double* q, const double* g, double lr, double* out, int B, cudaStream_t st) {
  step_kernel<<<(B + 127) / 128, 128, 0, st>>>(J, q, g, lr, out, B);
  return cudaGetLastError();
}

}  // namespace dgx

#ifdef DGX_PROFILE_REGIONS
extern "C" int dgx_prof_read(unsigned long long* out, int n, int reset) {
  if (n > 48) n = 48;
  cudaMemcpyFromSymbol(out, dgx::g_prof, sizeof(unsigned long long) * n);
  if (reset) {
    unsigned long long z[48] = {0};
    cudaMemcpyToSymbol(dgx::g_prof, z, sizeof z);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 101;
}
#endif
