// dgx_kernel.cuh — types shared by the fused kernel (dgx_kernels.cu) and the
// C-ABI implementation (dgx_capi.cu).
#pragma once

#include "dgx_geom.h"

namespace dgx {

constexpr int kMaxSims = 8;        // protocol velocities per candidate (standard: 7)
constexpr int kMaxDim = 32;        // 6 + J gradient coordinates (J <= 26)
constexpr int kSlotCap = 256;      // distinct active contacts per perturbation sim
constexpr int kStageDoubles = 640; // per-warp staging (adjoint segment: 4 slots x 5 x 32 lanes)

enum Mode : int { kModeGrad = 0, kModeEval = 1, kModeOpt = 2 };

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
  int f;      // flattened (sweep * N + point)
  int slot;
};

// One contact slot (sim.hpp:149-155) plus its friction replay data and the
// adjoints of its final lambda_n / n_world.
struct SlotRec {
  double lambda_n;
  double n[3];
  double rb[3];
  double fx[3];   // state before this slot's friction correction
  double fq[4];
  double a_lam;
  double a_n[3];
  int point;
  int last_corr;
  int fric;       // 1 if apply_friction changed the state
  int pad;
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
  V3 com;
  M3 inertia_body_inv;
};

struct KSim {
  double dt, mu, alpha, radius;
  int gs, M, measure_residual, pad;
  double vel[kMaxSims][3];
  double w_stable, w_qrange, w_qlimit;
};

struct KOpt {
  int iters, k_begin, k_end, record;
  double r0, lr, beta1, beta2, eps;
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
  CorrRec* corr;        // [grid, M, cap_corr]
  SlotRec* slots;       // [grid, M, kSlotCap]
  int cap_corr;
  int B;
};

// dynamic shared memory layout (bytes), identical on host and device
struct SmemLayout {
  int off_px, off_py, off_pz, off_link, off_ft, off_bitmap, off_slotpt, off_stage, off_misc, total;
  __host__ __device__ static int align(int x) { return (x + 15) & ~15; }
  __host__ __device__ SmemLayout(int N, int L, int M) {
    int o = 0;
    off_px = o; o = align(o + 8 * N);
    off_py = o; o = align(o + 8 * N);
    off_pz = o; o = align(o + 8 * N);
    off_link = o; o = align(o + 8 * 12 * L);
    off_ft = o; o = align(o + 8 * 6 * L * M);
    off_bitmap = o; o = align(o + 4 * ((N + 31) / 32) * M);
    off_slotpt = o; o = align(o + 4 * kSlotCap * M);
    off_stage = o; o = align(o + 8 * kStageDoubles * M);
    off_misc = o; o = align(o + 8 * (64 + 4 * kMaxDim + 2 * kMaxSims));
    total = o;
  }
};

}  // namespace dgx

#include <cuda_runtime.h>

namespace dgx {
cudaError_t launch_fused(const KHand& H, const KObj& O, int kind, const SphereSdf& sph, const BoxSdf& box,
                         const GridSdf& grd, const KSim& S, const KOpt& P, const KBuf& buf, int mode, int grid,
                         int smem, cudaStream_t st);
cudaError_t fused_occupancy(int kind, int M, int smem, int* blocks_per_sm);
cudaError_t launch_forward(const KHand& H, const double* q, double* out, int B, int grid, cudaStream_t st);
cudaError_t launch_step(int J, const double* q, const double* g, double lr, double* out, int B, cudaStream_t st);
}  // namespace dgx
