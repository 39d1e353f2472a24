// dgx_kernel.cuh — types shared by the fused kernel (dgx_kernels.cu) and the
// C-ABI implementation (dgx_capi.cu).
#pragma once

#include "dgx_mesh.h"

// Device-side bounds checks for the checked build (-DDGX_CHECKS, tools/
// build_checked.sh): every scratch / log / staging index against its
// capacity; a violation prints the site and traps. Compiled out otherwise.
#ifdef DGX_CHECKS
#include <cstdio>
#define DGX_ASSERT(c)                                                              \
  do {                                                                             \
    if (!(c)) {                                                                    \
      printf("DGX_ASSERT failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
             static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));          \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
#else
#define DGX_ASSERT(c) \
  do {                \
  } while (0)
#endif

namespace dgx {

constexpr int kMaxSims = 8;        // protocol velocities held inline in KSim (standard: 7); more: KSim::vel_dev
constexpr int kMaxWarps = 7;       // warps per grasp-search CTA: warp w runs sims w, w + W, ... (W = min(M, 7))
constexpr int kMaxDim = 32;        // 6 + J gradient coordinates (J <= 26)
constexpr int kSegMaxCap = 16;
constexpr int kCorrMatDoubles = 19 * 8 + 1;  // dgx_kernels.cu kCorrMat
// correction-reverse matrices are built kCorrBatch at a time, just before the
// reverse sweep reaches them, into a per-warp ring (L1 / L2-resident)
#ifndef DGX_CORR_BATCH
#define DGX_CORR_BATCH 16
#endif
constexpr int kCorrBatch = DGX_CORR_BATCH;
// lane adjoint (dgx_lane_adj.cuh): positions per step of a thread's reverse walk
// (independent geometry, then the serial recurrence); needs N >= kLaneU
#ifndef DGX_LANE_U
#define DGX_LANE_U 2  // config 3 (adjoint ms per 4096-candidate step): U 1 43.8, 2 30.9, 4 36.6, 8 85.3
#endif
constexpr int kLaneU = DGX_LANE_U;

enum Mode : int { kModeGrad = 0, kModeEval = 1, kModeOpt = 2 };

// Execution phases of one candidate-iteration (DESIGN.md §3 "split
// execution"): the fused kernel runs both halves in one warp per sim; the
// split pair runs the forward sweep at a higher occupancy (its register
// budget is not set by the adjoint) and hands over through FwdRec + the
// per-(candidate, sim) logs.
// kPhaseAdjTask: the split adjoint as independent warp tasks (one (candidate,
// sim) per task, points read from the forward's global copy, the candidate's
// epilogue run by the warp that finishes its last sim).
enum Phase : int { kPhaseFused = 0, kPhaseFwd = 1, kPhaseAdj = 2, kPhaseAdjTask = 3,
                   kPhaseFwdPtsG = 4 /* occupancy query only: the forward with global points */ };

enum Status : int {
  kOk = 0,
  kNonFiniteLoss = 1,
  kNonFiniteGrad = 2,
  kCorrOverflow = 3,
  kSlotOverflow = 4,
  kReplayMismatch = 5,
};

// One active Gauss-Seidel correction (sim.hpp:215-245): the state AFTER it.
struct CorrRec {
  double x[3];
  double q[4];
  double lam;
  // recorded values of the correcting point (sdf.cpp:83-107, sim.hpp:160-161)
  double g[3];      // grad_obj (recorded unit gradient)
  double rel[3];    // p - x before the correction
  double dx[3];     // r_local - proxy point
  double rho_d;     // dilated distance (C = -rho_d)
  double E[4];      // quat_exp(-lam * iwa)
  double sin_half;  // sin(|lam * iwa| / 2), 0 on the small-angle branch
  int f;            // flattened (sweep * N + point)
  int slot;
  int sign;         // PhongQuery::sign
  int fb;           // interpolated-normal fallback branch taken
};

// One contact slot (sim.hpp:149-155) plus its friction replay data and the
// adjoints of its final lambda_n / n_world.
struct SlotRec {
  double lambda_n;
  double n[3];
  double rb[3];
  double fx[3];   // state before this slot's friction correction
  double fq[4];
  double fE[4];   // friction's quat_exp(-lam_t * iwat) and its sin(half angle)
  double fsin;
  double a_lam;
  double a_n[3];
  int point;
  int last_corr;
  int fric;       // 1 if apply_friction changed the state
  int pad;
};

// Forward state handed from the forward kernel to the adjoint kernel, per
// (candidate, sim): the state after the solve (sim.hpp:188-196) and log sizes.
struct FwdRec {
  double x[3];
  double q[4];
  double residual;
  int ncorr, nslot, nfric, touched, status, pad;
};

// Per (warp slot, step) record of a multi-step perturbation sim
// (StabilityProtocol::steps > 1): the step's handover plus its prev / pred
// states and log offsets, for the reverse over the steps.
struct StepRec {
  FwdRec rec;
  double prev[13];  // x 3, q 4, xdot 3, thetadot 3
  double pred[13];
  int c_off, s_off, f_off, pad;
};

struct KHand {
  int L, J, N;
  const int* topo;
  const int* link_parent_joint;
  const int* joint_parent;
  const int* joint_child;
  const double* axis;
  const double* origin_R;
  const double* origin_t;
  const double* lower;
  const double* upper;
  const double* samples;      // [N*3]
  const int* sample_link;     // [N]
};

struct KObj {
  double mass;
  double inv_mass;        // 1.0 / mass (sim.hpp:141)
  V3 com;
  M3 inertia_body_inv;    // InertialData::inertia_body_inv (rigid.hpp:12)
  M3 Iw;                  // world_inertia_inv at the predicted pose (sim.hpp:96-100, 142)
};

struct KSim {
  double dt, mu, alpha, radius;
  int gs, M, measure_residual, seg_max;
  int steps, fold;         // fold: warp-task adjoint folds the identical final sweeps (exact)
  int pts_global;          // split forward: world points in buf.fk instead of shared memory
  int discard;             // drop consumed scratch lines from L2 without write-back (discard.global.L2)
  double vel[kMaxSims][3];
  const double* vel_dev;  // [M,3] device copy when M > kMaxSims
  double w_stable, w_qrange, w_qlimit;
  // grasp-energy terms (dgx_grasp_energy_batch; 0 = off)
  double w_fc, w_pen, fc_thr, fc_scale;
  __host__ __device__ int warps() const { return M < kMaxWarps ? M : kMaxWarps; }
};

struct KOpt {
  int iters, k_begin, k_end, record;
  double r0, lr, beta1, beta2, eps;
  int traj_k0, traj_rows;  // traj row of iterate k: b * traj_rows + (k - traj_k0)
};

struct KBuf {
  double* q;            // [B, 7+J] in (out for opt)
  double* adam_m;       // [B, D]
  double* adam_v;       // [B, D]
  double* losses;       // [B, 3]
  double* grads;        // [B, 3, D]  d_stable, d_qrange, d_qlimit
  double* stats;        // [B, M, 5]  SolveStats (eval)
  double* sim_res;      // [B, M]
  double* sim_grads;    // [B, M, D]   debug: per-perturbation gradient
  double* point_grads;  // [B, M, N, 3] debug: d residual_m / d p_i
  double* traj;         // [B, k_end-k_begin, 3 + D] opt: losses + weighted grad per iterate
  int* status;          // [B]
  const double* egrad;  // [B, D] opt: weighted grasp-energy gradient added before Adam (null: off)
  // warp-task adjoint (kPhaseAdjTask): per (candidate, sim) link sums, residual
  // and status, and per candidate the count of finished sims (zeroed per launch)
  double* task_ft;      // [B, M, 6L]
  double* task_res;     // [B, M]
  int* task_stat;       // [B, M]
  int* task_done;       // [B]
  StepRec* steps;       // [grid, W, T] multi-step sims (fused kernel, T > 1)
  CorrRec* corr;        // [grid, M, cap_corr]
  SlotRec* slots;       // [grid, M, N]  contact slots (one per hand point at most)
  int* slot_of_point;   // [grid, M, N]
  int* fric_order;      // [grid, M, N]
  FwdRec* fwd;          // [B, M] split execution only
  double* fk;           // [B, 12 L + 3 N] split: link transforms + world points of the forward
  int slot_stride;      // slots / fric_order entries per sim (N fused, cap_corr + 1 split)
  double* ft_global;    // [grid, M, L*6] adjoint link-sum spill buffers
  double* cmat;         // [grid, M, cap_corr, kCorrMat] batched correction reverse
  int* mesh_cache;      // [grid, M, gs*N] mesh objects: forward (face << 1 | inside) per point-sweep
  double* mesh_cert;    // [grid, M, N, 4] mesh objects: nearest-face certificate centre + radius
  int* mesh_cf;         // [grid, M, N, 1 + kCertFaces] certificate face sets
  int cap_corr;
  int B;
  // dynamic candidate claiming: each CTA takes blockIdx.x first, then tickets
  // from *claim (candidate = ticket + gridDim.x); the counter is zeroed on the
  // stream before every launch. null = static stride (DGX_STATIC_SCHED)
  unsigned long long* claim;
};

// warp-task adjoint: warps per CTA and the per-warp shared memory (doubles):
// adjoint staging (also the epilogue's copy of the candidate's per-sim link
// sums + scratch), link sums of the running sim, configuration, gradients
#ifndef DGX_TASK_WARPS
#define DGX_TASK_WARPS 8
#endif
constexpr int kTaskWarps = DGX_TASK_WARPS;
constexpr int kTaskRing = 8;  // candidate slots a task CTA can have in flight
struct TaskLayout {
  int stage, off_ft, off_sq, off_sg, per_warp;
  __host__ __device__ TaskLayout(int L, int M, int seg_max) {
    const int a = seg_max * 5 * 32, b2 = (M + 1) * 6 * L + 2 * M + 8;
    stage = a > b2 ? a : b2;
    off_ft = stage;
    off_sq = off_ft + 6 * L;
    off_sg = off_sq + 40;
    per_warp = off_sg + 3 * 32;
  }
  // + the CTA's task queue: next task, ring of (slot tag | candidate), per-slot resolved counts
  __host__ __device__ int bytes() const { return 8 * per_warp * kTaskWarps + 16 + 8 * kTaskRing + 4 * kTaskRing; }
};

// dynamic shared memory layout (bytes), identical on host and device. Per
// sim: link force / torque sums (ft) and residuals; per warp: bitmap and
// adjoint staging (a warp runs sims warp, warp + W, ...).
struct SmemLayout {
  int off_px, off_py, off_pz, off_link, off_ft, off_bitmap, off_stage, off_misc, off_sres, off_sflag, total;
  __host__ __device__ static int align(int x) { return (x + 15) & ~15; }
  int stage_per_warp;  // doubles: seg_max x 5 x 32 adjoint staging (>= 6L + kMaxDim for the debug FK adjoint)
  __host__ __device__ static int stage_doubles(int seg_max, int L) {
    const int a = seg_max * 5 * 32, b = 6 * L + kMaxDim;
    return a > b ? a : b;
  }
  __host__ __device__ SmemLayout(int N, int L, int M, int seg_max, bool points = true) {
    stage_per_warp = stage_doubles(seg_max, L);
    const int W = M < kMaxWarps ? M : kMaxWarps;
    const int np = points ? N : 0;
    int o = 0;
    off_px = o; o = align(o + 8 * np);
    off_py = o; o = align(o + 8 * np);
    off_pz = o; o = align(o + 8 * np);
    off_link = o; o = align(o + 8 * 12 * L);
    off_ft = o; o = align(o + 8 * 6 * L * M);
    off_bitmap = o; o = align(o + 4 * ((N + 31) / 32) * W);
    off_stage = o; o = align(o + 8 * stage_per_warp * W);
    off_misc = o; o = align(o + 8 * (40 + 3 * kMaxDim + 8));  // q, 3 gradients, next-candidate slot
    off_sres = o; o = align(o + 8 * M);
    off_sflag = o; o = align(o + 4 * (M + 1));                 // per-sim status, [M] = candidate status
    total = o;
  }
};

}  // namespace dgx

#include <cuda_runtime.h>

namespace dgx {
// one object's SDF backend; `kind` selects the member
struct SdfSet {
  int kind;
  SphereSdf sph;
  BoxSdf box;
  GridSdf grd;
  MeshSdf mesh;
};
// phase: kPhaseFused (any backend) or kPhaseFwd / kPhaseAdj (analytic and grid
// backends; see split_capable)
cudaError_t launch_fused(const KHand& H, const KObj& O, const SdfSet& sdf, const KSim& S, const KOpt& P,
                         const KBuf& buf, int mode, int phase, int grid, int smem, cudaStream_t st);
cudaError_t fused_occupancy(int kind, int M, int smem, int phase, int* blocks_per_sm);
// split adjoint as warp tasks (analytic and grid backends); grid = #SM x occupancy
cudaError_t launch_adj_task(const KHand& H, const KObj& O, const SdfSet& sdf, const KSim& S, const KOpt& P,
                            const KBuf& buf, int mode, int grid, int smem, cudaStream_t st);
cudaError_t adj_task_occupancy(int kind, int smem, int* per_sm);
// split adjoint with one thread per (candidate, sim) (dgx_lane_adj.cuh), then
// the per-candidate epilogue kernel (one warp per candidate)
cudaError_t launch_lane_adj(const KHand& H, const KObj& O, const SdfSet& sdf, const KSim& S, const KOpt& P,
                            const KBuf& buf, int mode, cudaStream_t st);
cudaError_t launch_lane_epi(const KHand& H, const KSim& S, const KOpt& P, const KBuf& buf, int mode, cudaStream_t st);
inline bool split_capable(int kind) { return kind != kSdfMesh; }
// out[n, 8] = rho - radius, grad (3), proxy (3), sign per point (MeshSdf::dilated,
// sdf.cpp:62-67); within != 0: dilated_within (sdf.cpp:69-81), culled points
// report sign 0 and rho = +inf
cudaError_t launch_sdf_query(const SdfSet& sdf, int n, const double* r, double radius, int within, double* out,
                             cudaStream_t st);
cudaError_t launch_forward(const KHand& H, const double* q, double* out, int B, int grid, cudaStream_t st);
cudaError_t launch_contacts(const KHand& H, const SdfSet& sdf, int B, const double* q, const double* area, int T,
                            const double* thr, int cap, double* ca, int* cnt, int* ncont, int* cidx, double* crec,
                            int grid, cudaStream_t st);
// grasp-energy terms (dgx_grasp_energy_batch): e [B,2], g [B,2,D], gw [B,D]
// (each may be null); candidates with status != 0 are skipped (status may be null)
cudaError_t launch_energy(const KHand& H, const KObj& O, const SdfSet& sdf, const KSim& S, int B, const double* q,
                          const int* status, double* e, double* g, double* gw, int grid, cudaStream_t st);
cudaError_t launch_step(int J, const double* q, const double* g, double lr, double* out, int B, cudaStream_t st);
}  // namespace dgx
