// dgx_capi.cu — implementation of include/dgx.h over the sm_100a kernels.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <limits>
#include <vector>

#include "../../include/dgx.h"
#include "dgx_kernel.cuh"
#include "dgx_mesh_host.h"
#include "dgx_drop.cuh"

using namespace dgx;

namespace {

thread_local std::string g_err;

struct DgxError : std::runtime_error {
  int code;
  DgxError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DgxError(DGX_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return DGX_OK;
  } catch (const DgxError& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DGX_E_INVALID;
  }
}

struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  void ensure(size_t bytes) {
    if (bytes <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cuda_check(cudaMalloc(&p, bytes), "cudaMalloc");
    n = bytes;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

}  // namespace

// per-stream kernel scratch (correction logs, contact slots, link-sum spills)
struct Scratch {
  DevBuf corr, slots, ftg, mcache, drop, thr, claim, vel, egrad;
  void release() {
    claim.release();
    vel.release();
    egrad.release();
    thr.release();
    corr.release();
    slots.release();
    ftg.release();
    mcache.release();
    drop.release();
  }
};

// a side stream with its own scratch, for concurrent per-object launches
struct SubStream {
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
  Scratch scratch;
};

struct dgx_ctx {
  int device = 0;
  int num_sms = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr;
  int cap_corr = 1024;
  int adjoint = DGX_ADJOINT_AUTO;  // dgx_ctx_set_adjoint
  int64_t launches = 0;
  // kernel timing (dgx_ctx_set_kernel_timing): event pairs per launch
  bool timing = false;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> timed;  // kind, (start, stop)
  std::vector<cudaEvent_t> event_pool;
  Scratch scratch;
  DevBuf io;
  std::vector<SubStream> subs;
};

struct dgx_hand {
  dgx_ctx* ctx;
  int L, J, N;
  DevBuf mem;
  KHand k;
  std::vector<double> lower, upper;
};

struct dgx_object {
  dgx_ctx* ctx;
  int kind;
  SdfSet sdf{};
  DevBuf vals;  // grid values, or the mesh block (nodes, faces, tri, vx, vn, MeshGeom)
  DevBuf bmin;  // grids: block lower bounds of the forward pre-filter (GridSdf::bmin)
  KObj k;
  // mesh objects: device vertices + count (table-contact samples of the drop)
  const double* mesh_vx = nullptr;
  int mesh_nv = 0;
  M3 inertia_body{};
  bool has_inertia_body = false;
};

namespace {

void set_device(dgx_ctx* c) { cuda_check(cudaSetDevice(c->device), "cudaSetDevice"); }

KSim make_sim(const dgx_params* p, bool eval) {
  if (!p) throw DgxError(DGX_E_INVALID, "params is NULL");
  if (p->steps < 1) throw DgxError(DGX_E_INVALID, "StabilityProtocol::steps must be >= 1");
  if (p->num_velocities < 1) throw DgxError(DGX_E_INVALID, "protocol must have >= 1 velocities");
  if (p->num_velocities > kMaxSims && !p->velocity_list)
    throw DgxError(DGX_E_INVALID, "more than 8 velocities need params->velocity_list");
  if (p->gs_iters < 0) throw DgxError(DGX_E_INVALID, "gs_iters must be >= 0");
  if (p->dilation_radius < 0.0) throw std::invalid_argument("dilation radius must be >= 0");
  if (!(p->dt > 0.0)) throw DgxError(DGX_E_INVALID, "dt must be > 0");
  if (!(p->w_force_closure >= 0.0) || !(p->w_penetration >= 0.0))
    throw DgxError(DGX_E_INVALID, "grasp-energy weights must be >= 0");
  KSim s{};
  s.dt = p->dt;
  s.mu = p->mu;
  s.alpha = p->alpha_leak;
  s.radius = p->dilation_radius;
  s.gs = p->gs_iters;
  s.M = p->num_velocities;
  s.steps = p->steps;
  s.measure_residual = eval ? 1 : 0;
  for (int m = 0; m < s.M && m < kMaxSims; ++m)
    for (int c = 0; c < 3; ++c) s.vel[m][c] = p->velocity_list ? p->velocity_list[3 * m + c] : p->velocities[m][c];
  s.vel_dev = nullptr;  // set by upload_velocities when M > kMaxSims
  s.discard = std::getenv("DGX_NO_DISCARD") ? 0 : 1;
  s.w_stable = p->w_stable;
  s.w_qrange = p->w_qrange;
  s.w_qlimit = p->w_qlimit;
  s.w_fc = p->w_force_closure;
  s.w_pen = p->w_penetration;
  s.fc_thr = p->contact_threshold > 0.0 ? p->contact_threshold : 0.005;
  s.fc_scale = p->torque_scale > 0.0 ? p->torque_scale : 0.05;
  return s;
}

// M > kMaxSims: the velocity list goes to device memory, stream-ordered on the
// context stream (pageable source: staged before cudaMemcpyAsync returns)
void upload_velocities(dgx_ctx* c, KSim& S, const dgx_params* p) {
  if (S.M <= kMaxSims) return;
  if (!c) throw DgxError(DGX_E_INVALID, "NULL context");
  set_device(c);
  c->scratch.vel.ensure(sizeof(double) * 3 * S.M);
  cuda_check(cudaMemcpyAsync(c->scratch.vel.p, p->velocity_list, sizeof(double) * 3 * S.M, cudaMemcpyHostToDevice,
                             c->stream),
             "H2D velocities");
  S.vel_dev = static_cast<const double*>(c->scratch.vel.p);
}

bool energy_on(const KSim& S) { return S.w_fc != 0.0 || S.w_pen != 0.0; }

// adjoint staging length S.seg_max; returns the adjoint kernel's shared memory
int choose_staging(const dgx_hand* h, const dgx_object* o, KSim& S) {
  const int M = S.M;
  // longest adjoint segment whose staging still fits one CTA's shared memory
  S.seg_max = 0;
  // Adjoint staging length (points per lane): the longest up to 12 whose
  // shared memory stays within the 196 KB carve-out tier (1 KB is reserved per
  // CTA), so >= 60 KB of L1 remain for the SDF data. Config 2 (allegro16,
  // 40-step bench, candidate-iterations/s): seg 16 needs 197.5 KB -> the 228 KB
  // tier, ~28 KB of L1 -> 71k; seg 12-14 -> 78-79k; seg 15 -> 77k; seg 8 ->
  // 77k; seg 4 -> 72k. Larger hands fall back to the longest staging that fits
  // at all. Mesh objects run two CTAs per SM (dgx_kernels.cu CtasPerSm) and
  // cap it at 4.
  int seg_cap = o->kind == DGX_SDF_MESH ? 4 : 12;
  if (const char* ev = std::getenv("DGX_SEGMAX")) seg_cap = std::max(1, std::min(kSegMaxCap, std::atoi(ev)));
  for (int limit : {195 * 1024, 227 * 1024}) {
    for (int seg = seg_cap; seg >= 1 && S.seg_max == 0; --seg)
      if (SmemLayout(h->N, h->L, M, seg).total <= limit) S.seg_max = seg;
    if (S.seg_max) break;
  }
  if (S.seg_max == 0)
    throw DgxError(DGX_E_UNSUPPORTED, "hand too large for one CTA's shared memory (N=" + std::to_string(h->N) + ")");
  return SmemLayout(h->N, h->L, M, S.seg_max).total;
}

// grid of persistent CTAs and the scratch it needs (fused execution)
int prepare(dgx_ctx* c, Scratch& sc, const dgx_hand* h, const dgx_object* o, KSim& S, int B, KBuf& buf,
            int& smem) {
  const int M = S.M;
  smem = choose_staging(h, o, S);
  int per_sm = 0;
  cuda_check(fused_occupancy(o->kind, M, smem, kPhaseFused, &per_sm), "occupancy");
  if (per_sm < 1) throw DgxError(DGX_E_UNSUPPORTED, "fused kernel cannot be resident (registers/smem)");
  int grid = c->num_sms * per_sm;
  if (grid > B) grid = B;
  if (grid < 1) grid = 1;
  const size_t nws = static_cast<size_t>(grid) * M;
  sc.corr.ensure(nws * c->cap_corr * sizeof(CorrRec));
  const size_t per = nws * static_cast<size_t>(h->N);
  // contact slots: one per hand point per solve (sim.hpp:155); a multi-step
  // protocol keeps every step's slots (nslot <= ncorr + T overall)
  const int T = S.steps;
  const size_t ss = T > 1 ? std::max<size_t>(h->N, static_cast<size_t>(c->cap_corr) + T) : h->N;
  const size_t steps_bytes = T > 1 ? nws * T * sizeof(StepRec) + 256 : 0;
  sc.slots.ensure(nws * ss * (sizeof(SlotRec) + sizeof(int)) + per * sizeof(int) + steps_bytes + 256);
  buf.corr = static_cast<CorrRec*>(sc.corr.p);
  buf.slots = static_cast<SlotRec*>(sc.slots.p);
  buf.slot_of_point = reinterpret_cast<int*>(buf.slots + nws * ss);
  buf.fric_order = buf.slot_of_point + per;
  buf.slot_stride = static_cast<int>(ss);
  buf.steps = T > 1 ? reinterpret_cast<StepRec*>((reinterpret_cast<uintptr_t>(buf.fric_order + nws * ss) + 255) &
                                                 ~static_cast<uintptr_t>(255))
                    : nullptr;
  buf.fwd = nullptr;
  buf.fk = nullptr;
  sc.ftg.ensure(nws * (6 * static_cast<size_t>(h->L) + static_cast<size_t>(kCorrBatch) * kCorrMatDoubles) *
                sizeof(double));
  buf.ft_global = static_cast<double*>(sc.ftg.p);
  buf.cmat = buf.ft_global + nws * 6 * static_cast<size_t>(h->L);
  buf.mesh_cache = nullptr;
  buf.mesh_cert = nullptr;
  buf.mesh_cf = nullptr;
  if (o->kind == DGX_SDF_MESH) {
    // per point-sweep (face, sign) of the forward, read by the adjoint; per
    // point nearest-face certificates (4 doubles + 1 + kCertFaces ints)
    const size_t b_cache =
        (per * static_cast<size_t>(std::max(S.gs, 1)) * static_cast<size_t>(T) * sizeof(int) + 255) & ~size_t(255);
    const size_t b_cert = (per * 4 * sizeof(double) + 255) & ~size_t(255);
    sc.mcache.ensure(b_cache + b_cert + per * (kCertFaces + 1) * sizeof(int));
    char* base = static_cast<char*>(sc.mcache.p);
    buf.mesh_cache = reinterpret_cast<int*>(base);
    buf.mesh_cert = reinterpret_cast<double*>(base + b_cache);
    buf.mesh_cf = reinterpret_cast<int*>(base + b_cache + b_cert);
  }
  buf.cap_corr = c->cap_corr;
  buf.B = B;
  return grid;
}

// Split execution for the analytic and grid backends: per
// chunk of candidates the forward kernel (kFwdCtasPerSm CTAs per SM: its
// register budget is not set by the adjoint) and then the adjoint kernel,
// handing over through FwdRec and per-(candidate, sim) logs. Mesh objects run
// fused. DGX_FUSED=1 forces the fused kernel everywhere (A/B measurements).
bool use_split(const dgx_object* o) {
  static const bool fused_env = std::getenv("DGX_FUSED") != nullptr;
  return split_capable(o->kind) && !fused_env;
}

constexpr size_t kSplitScratchBytes = size_t(8) << 30;  // per stream
constexpr size_t kLaneScratchBytes = size_t(24) << 30;  // per stream, lane adjoint
constexpr int kSplitMaxFwdSmem = 96 * 1024;

struct SplitGrid {
  int chunk, grid_f, grid_a, smem_f, smem_a;
  bool task;  // adjoint as warp tasks (adj_task_kernel) instead of one CTA per candidate
  bool lane;  // adjoint with one thread per (candidate, sim) + the epilogue kernel (the default)
};

// Split adjoint variant. Default (auto): the lane adjoint
// (lane_adj_kernel, one thread per (candidate, sim), dgx_lane_adj.cuh) when the
// batch gives it at least kLaneMinWarpsPerSm warps per SM, else the CTA-per-
// candidate adjoint (bit-identical to the fused kernel). The lane adjoint's
// parallelism is its task count. Config-3 workload, whole step cand-iter/s
// lane vs CTA (tools/adjoint_crossover.sh): 1024 candidates (1.5 warps / SM)
// 35.6k vs 57.8k, 2048 (3 warps / SM) 64.5k vs 60.5k, 3072 80.4k vs 57.7k,
// 4096 (6 warps / SM) 97.7k vs 55.8k. DGX_ADJ=lane|cta|task forces one (A/B
// measurements); DGX_ADJ_TASK=1 is the warp-task adjoint (never faster).
constexpr int kLaneMinWarpsPerSm = 3;
int adjoint_variant() {  // 0 cta, 1 task, 2 lane, 3 auto
  static const int v = [] {
    const char* ev = std::getenv("DGX_ADJ");
    if (std::getenv("DGX_ADJ_TASK")) return 1;
    if (!ev) return 3;
    if (std::strcmp(ev, "cta") == 0) return 0;
    if (std::strcmp(ev, "task") == 0) return 1;
    if (std::strcmp(ev, "lane") == 0) return 2;
    return 3;
  }();
  return v;
}

// Split adjoint as warp tasks (DGX_ADJ_TASK=1; measured equal to the CTA-per-
// candidate adjoint on configs 2 and 3, so the CTA adjoint,
// bit-identical to the fused kernel, stays the default). Its staging length:
// DGX_TASK_SEG (default 8 points per lane: 8 warps x 11.5 KB leave most of the
// SM's 256 KB as L1 for the points and SDF cells the tasks read from L2).
int task_seg() {
  static const int seg = [] {
    const char* ev = std::getenv("DGX_TASK_SEG");
    return ev ? std::max(1, std::min(kSegMaxCap, std::atoi(ev))) : 8;
  }();
  return seg;
}

// concurrent: how many such launches run at once on side streams
// (dgx_optimize_multi); the lane adjoint's parallelism is their summed tasks
SplitGrid prepare_split(dgx_ctx* c, Scratch& sc, const dgx_hand* h, const dgx_object* o, KSim& S, int B,
                        bool record, KBuf& buf, int concurrent) {
  const int M = S.M, N = h->N, L = h->L;
  SplitGrid g{};
  int av = adjoint_variant();
  if (av == 3 && c->adjoint != DGX_ADJOINT_AUTO) av = c->adjoint == DGX_ADJOINT_LANE ? 2 : 0;
  g.task = record && av == 1;
  g.lane = record && N >= 64 &&  // (the lane adjoint stages blocks of <= 64 positions)
           (av == 2 || (av == 3 && static_cast<long long>(B) * M * std::max(1, concurrent) >=
                                       static_cast<long long>(kLaneMinWarpsPerSm) * 32 * c->num_sms));
  if (g.lane) {
    g.smem_a = 0;
  } else if (g.task) {
    S.seg_max = task_seg();
    S.fold = std::getenv("DGX_NOFOLD") ? 0 : 1;
    g.smem_a = TaskLayout(L, M, S.seg_max).bytes();
  } else {
    g.smem_a = choose_staging(h, o, S);
  }
  g.smem_f = SmemLayout(N, L, M, 0, !S.pts_global).total;
  int per_f = 0, per_a = 1;
  cuda_check(fused_occupancy(o->kind, M, g.smem_f, S.pts_global ? kPhaseFwdPtsG : kPhaseFwd, &per_f), "occupancy");
  if (record) {
    if (g.lane) per_a = 1;
    else if (g.task) cuda_check(adj_task_occupancy(o->kind, g.smem_a, &per_a), "occupancy");
    else cuda_check(fused_occupancy(o->kind, M, g.smem_a, kPhaseAdj, &per_a), "occupancy");
  }
  if (per_f < 1 || per_a < 1) throw DgxError(DGX_E_UNSUPPORTED, "split kernels cannot be resident (registers/smem)");
  g.grid_f = c->num_sms * per_f;
  g.grid_a = c->num_sms * per_a;
  // logs live per (candidate, sim) for one chunk: ~(cap_corr + 1) x 372 B + 8 N B per sim. Chunks
  // are as large as kSplitScratchBytes allows (each chunk boundary drains both kernels' tails);
  // DGX_SPLIT_SCRATCH_MB lowers the budget, down to 4 waves of the larger grid per chunk.
  const size_t per_cand = static_cast<size_t>(M) * ((static_cast<size_t>(c->cap_corr) + 1) *
                                                        (sizeof(CorrRec) + sizeof(SlotRec) + sizeof(int)) +
                                                    sizeof(FwdRec) + static_cast<size_t>(N) * sizeof(int) +
                                                    (6 * static_cast<size_t>(L) + 2) * sizeof(double)) +
                          (12 * static_cast<size_t>(h->L) + 3 * static_cast<size_t>(N)) * sizeof(double) + 8;
  // the lane adjoint's parallelism is its task count (one thread per (candidate,
  // sim)): it takes the whole batch in one chunk when kLaneScratchBytes allows
  size_t budget = g.lane ? kLaneScratchBytes : kSplitScratchBytes;
  if (const char* ev = std::getenv("DGX_LANE_SCRATCH_MB"); ev && g.lane)
    budget = static_cast<size_t>(std::max(1, std::atoi(ev))) << 20;
  if (const char* ev = std::getenv("DGX_SPLIT_SCRATCH_MB"))  // tests: force several chunks
    budget = static_cast<size_t>(std::max(1, std::atoi(ev))) << 20;
  const size_t by_mem = std::max<size_t>(1, budget / per_cand);
  g.chunk = static_cast<int>(std::max<size_t>(
      1, std::min<size_t>(B, std::max<size_t>(4 * static_cast<size_t>(std::max(g.grid_f, g.grid_a)), by_mem))));
  {  // equal chunks (4096 -> 2 x 2048, not 2973 + 1123): the same launch count, balanced launches
    const int n = (B + g.chunk - 1) / g.chunk;
    g.chunk = (B + n - 1) / n;
  }
  g.grid_f = std::min(g.grid_f, g.chunk);
  g.grid_a = std::min(g.grid_a, g.chunk);
  const size_t nws = static_cast<size_t>(g.chunk) * M;
  const size_t cap = static_cast<size_t>(c->cap_corr), ss = cap + 1;  // nslot <= ncorr <= cap_corr
  sc.corr.ensure(nws * cap * sizeof(CorrRec));
  const size_t fk_per = 12 * static_cast<size_t>(h->L) + 3 * static_cast<size_t>(N);
  const size_t task_bytes = nws * (6 * static_cast<size_t>(L) + 1) * sizeof(double) + nws * sizeof(int) +
                            static_cast<size_t>(g.chunk) * sizeof(int) + 3 * 256;
  sc.slots.ensure(nws * (ss * sizeof(SlotRec) + sizeof(FwdRec) + (ss + N) * sizeof(int)) +
                  static_cast<size_t>(g.chunk) * fk_per * sizeof(double) + 256 + task_bytes);
  char* base = static_cast<char*>(sc.slots.p);
  buf.corr = static_cast<CorrRec*>(sc.corr.p);
  buf.slots = reinterpret_cast<SlotRec*>(base);
  buf.fwd = reinterpret_cast<FwdRec*>(base + nws * ss * sizeof(SlotRec));
  buf.slot_of_point = reinterpret_cast<int*>(buf.fwd + nws);
  buf.fric_order = buf.slot_of_point + nws * N;
  buf.fk = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(buf.fric_order + nws * ss) + 255) & ~static_cast<uintptr_t>(255));
  buf.slot_stride = static_cast<int>(ss);
  {  // warp-task adjoint rows (per (candidate, sim)) and per-candidate counters
    auto al = [](void* p) {
      return reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(p) + 255) & ~static_cast<uintptr_t>(255));
    };
    char* tb = al(buf.fk + static_cast<size_t>(g.chunk) * fk_per);
    buf.task_ft = reinterpret_cast<double*>(tb);
    buf.task_res = buf.task_ft + nws * 6 * static_cast<size_t>(L);
    buf.task_stat = reinterpret_cast<int*>(al(buf.task_res + nws));
    buf.task_done = reinterpret_cast<int*>(al(buf.task_stat + nws));
  }
  // adjoint spill / correction-matrix buffers per resident warp
  const size_t nwa = g.task ? static_cast<size_t>(g.grid_a) * kTaskWarps : static_cast<size_t>(g.grid_a) * M;
  sc.ftg.ensure(nwa * (6 * static_cast<size_t>(h->L) + static_cast<size_t>(kCorrBatch) * kCorrMatDoubles) *
                sizeof(double));
  buf.ft_global = static_cast<double*>(sc.ftg.p);
  buf.cmat = buf.ft_global + nwa * 6 * static_cast<size_t>(h->L);
  buf.mesh_cache = nullptr;
  buf.mesh_cert = nullptr;
  buf.mesh_cf = nullptr;
  buf.cap_corr = c->cap_corr;
  return g;
}

cudaEvent_t pool_event(dgx_ctx* c) {
  if (!c->event_pool.empty()) {
    cudaEvent_t e = c->event_pool.back();
    c->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cuda_check(cudaEventCreate(&e), "cudaEventCreate");
  return e;
}

// one grasp-search launch of kind `phase` on st (counted; timed when enabled)
template <class F>
void counted_launch(dgx_ctx* c, int phase, cudaStream_t st, const char* what, F&& launch) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->timing) {
    e0 = pool_event(c);
    e1 = pool_event(c);
    cuda_check(cudaEventRecord(e0, st), "cudaEventRecord");
  }
  (void)cudaGetLastError();  // a stale non-sticky error must not be reported as this launch's
  cuda_check(launch(), what);
  ++c->launches;
  if (c->timing) {
    cuda_check(cudaEventRecord(e1, st), "cudaEventRecord");
    c->timed.push_back({phase, {e0, e1}});
  }
}

// Dynamic candidate claiming (next_candidate, dgx_kernels.cu). Every launch is
// self-contained: its ticket counter is zeroed on the launch stream right
// before it, so no host-side ticket base can drift from the device counter (a
// failed or partial earlier launch, a stale error, or another stream cannot
// skew later launches). DGX_STATIC_SCHED=1 keeps the static stride (A/B
// measurements).
void bind_claim(Scratch& sc, KBuf& buf, int, cudaStream_t st) {
  static const bool static_sched = std::getenv("DGX_STATIC_SCHED") != nullptr;
  if (static_sched) {
    buf.claim = nullptr;
    return;
  }
  sc.claim.ensure(sizeof(unsigned long long));
  cuda_check(cudaMemsetAsync(sc.claim.p, 0, sizeof(unsigned long long), st), "cudaMemsetAsync");
  buf.claim = static_cast<unsigned long long*>(sc.claim.p);
}

// Every launch for B candidates whose per-candidate arrays start at buf's
// pointers, on stream st with scratch sc.
void launch_range(dgx_ctx* c, Scratch& sc, const dgx_hand* h, const dgx_object* o, KSim S, KOpt P, KBuf buf,
                  int B, int mode, cudaStream_t st, int concurrent = 1) {
  const int M = S.M, D = 6 + h->J, Qd = 7 + h->J, N = h->N;
  if (mode == kModeOpt) {
    P.traj_k0 = P.k_begin;
    P.traj_rows = P.k_end - P.k_begin;
  }
  // Fused instead of split when the split cannot gain (measured):
  // * B <= #SMs: every candidate has an SM to itself in the fused kernel, and
  //   the split's per-iterate launches only cost (config 1: 61.5k vs 69.4k);
  // * forward shared memory > kSplitMaxFwdSmem (N >~ 3000 points): two forward
  //   CTAs leave too little L1 for the SDF cells (config 3, N = 4093: 42.9k vs 45.8k).
  // Large hands (forward shared memory with the points > kSplitMaxFwdSmem,
  // N >~ 3000) run the forward with its points in global memory (L1 / L2)
  // so it keeps two CTAs per SM (fwd_kernel<Sdf, true>).
  const bool split = use_split(o) && B > c->num_sms && !(mode == kModeOpt && P.k_end == P.k_begin) &&
                     S.steps == 1;  // multi-step protocols run the fused kernel
  S.pts_global = SmemLayout(N, h->L, M, 0).total > kSplitMaxFwdSmem ? 1 : 0;
  if (const char* ev = std::getenv("DGX_PTS_GLOBAL")) S.pts_global = std::atoi(ev) != 0;  // A/B
  // grasp-energy terms (optimizer only): their weighted gradient depends on
  // the iterate's q, so it is computed per iterate right before the
  // iterate's grasp-search launch and added before Adam (KBuf::egrad)
  const bool energy = mode == kModeOpt && energy_on(S);
  auto energy_launch = [&](const KBuf& cb, int nb, int k) {
    sc.egrad.ensure(sizeof(double) * static_cast<size_t>(nb) * D);
    (void)cudaGetLastError();
    cuda_check(launch_energy(h->k, o->k, o->sdf, S, nb, cb.q, k > P.traj_k0 ? cb.status : nullptr, nullptr,
                             nullptr, static_cast<double*>(sc.egrad.p), std::min(nb, c->num_sms * 4), st),
               "energy_kernel");
    ++c->launches;
  };
  if (!split) {
    int smem = 0;
    const int grid = prepare(c, sc, h, o, S, B, buf, smem);
    if (!energy) {
      bind_claim(sc, buf, B, st);
      counted_launch(c, kPhaseFused, st, "fused_kernel",
                     [&] { return launch_fused(h->k, o->k, o->sdf, S, P, buf, mode, kPhaseFused, grid, smem, st); });
      return;
    }
    for (int k = P.k_begin; k < P.k_end; ++k) {  // one fused launch per iterate
      KOpt Pk = P;
      Pk.k_begin = k;
      Pk.k_end = k + 1;
      energy_launch(buf, B, k);
      KBuf kb = buf;
      kb.egrad = static_cast<const double*>(sc.egrad.p);
      bind_claim(sc, kb, B, st);
      counted_launch(c, kPhaseFused, st, "fused_kernel",
                     [&] { return launch_fused(h->k, o->k, o->sdf, S, Pk, kb, mode, kPhaseFused, grid, smem, st); });
    }
    return;
  }
  const bool record = mode != kModeEval;
  const SplitGrid g = prepare_split(c, sc, h, o, S, B, record, buf, concurrent);
  const int k0 = mode == kModeOpt ? P.k_begin : 0, k1 = mode == kModeOpt ? P.k_end : 1;
  for (int b0 = 0; b0 < B; b0 += g.chunk) {
    const int nb = std::min(g.chunk, B - b0);
    const size_t o0 = static_cast<size_t>(b0);
    auto off = [&](auto* p, size_t per) { return p ? p + o0 * per : p; };
    KBuf cb = buf;
    cb.B = nb;
    cb.q = off(buf.q, Qd);
    cb.adam_m = off(buf.adam_m, D);
    cb.adam_v = off(buf.adam_v, D);
    cb.losses = off(buf.losses, 3);
    cb.grads = off(buf.grads, 3 * static_cast<size_t>(D));
    cb.stats = off(buf.stats, static_cast<size_t>(M) * 5);
    cb.sim_res = off(buf.sim_res, M);
    cb.sim_grads = off(buf.sim_grads, static_cast<size_t>(M) * D);
    cb.point_grads = off(buf.point_grads, static_cast<size_t>(M) * N * 3);
    cb.traj = off(buf.traj, static_cast<size_t>(P.traj_rows) * (3 + D));
    cb.status = off(buf.status, 1);
    for (int k = k0; k < k1; ++k) {
      KOpt Pk = P;
      if (mode == kModeOpt) {
        Pk.k_begin = k;
        Pk.k_end = k + 1;
      }
      if (energy) {
        energy_launch(cb, nb, k);
        cb.egrad = static_cast<const double*>(sc.egrad.p);
      }
      bind_claim(sc, cb, nb, st);
      counted_launch(c, kPhaseFwd, st, "forward kernel", [&] {
        return launch_fused(h->k, o->k, o->sdf, S, Pk, cb, mode, kPhaseFwd, std::min(g.grid_f, nb), g.smem_f, st);
      });
      if (!record) continue;
      bind_claim(sc, cb, nb, st);
      if (g.lane) {
        counted_launch(c, kPhaseAdj, st, "lane adjoint kernels", [&] {
          cudaError_t e = launch_lane_adj(h->k, o->k, o->sdf, S, Pk, cb, mode, st);
          if (e != cudaSuccess) return e;
          ++c->launches;  // + the epilogue kernel
          return launch_lane_epi(h->k, S, Pk, cb, mode, st);
        });
      } else if (g.task) {
        cuda_check(cudaMemsetAsync(cb.task_done, 0, sizeof(int) * nb, st), "cudaMemsetAsync");
        const int grid_t = std::max(1, std::min(g.grid_a, (nb * M + kTaskWarps - 1) / kTaskWarps));
        counted_launch(c, kPhaseAdj, st, "adjoint task kernel", [&] {
          return launch_adj_task(h->k, o->k, o->sdf, S, Pk, cb, mode, grid_t, g.smem_a, st);
        });
      } else {
        counted_launch(c, kPhaseAdj, st, "adjoint kernel", [&] {
          return launch_fused(h->k, o->k, o->sdf, S, Pk, cb, mode, kPhaseAdj, std::min(g.grid_a, nb), g.smem_a, st);
        });
      }
    }
  }
}

// host <-> device staging for non-device-pointer calls
struct Staging {
  dgx_ctx* c;
  bool dev;
  std::vector<std::pair<void*, std::pair<const void*, size_t>>> back;  // host dst, dev src, bytes
  size_t off = 0;
  explicit Staging(dgx_ctx* ctx, bool device_ptrs, size_t total) : c(ctx), dev(device_ptrs) {
    if (!dev) c->io.ensure(total + 256 * 16);
  }
  template <class T>
  T* in(const T* host, size_t count) {
    if (dev || !host) return const_cast<T*>(host);
    T* d = reinterpret_cast<T*>(static_cast<char*>(c->io.p) + off);
    off += (count * sizeof(T) + 255) & ~size_t(255);
    cuda_check(cudaMemcpyAsync(d, host, count * sizeof(T), cudaMemcpyHostToDevice, c->stream), "H2D");
    return d;
  }
  template <class T>
  T* out(T* host, size_t count, bool copy_in = false) {
    if (dev || !host) return host;
    T* d = reinterpret_cast<T*>(static_cast<char*>(c->io.p) + off);
    off += (count * sizeof(T) + 255) & ~size_t(255);
    if (copy_in) cuda_check(cudaMemcpyAsync(d, host, count * sizeof(T), cudaMemcpyHostToDevice, c->stream), "H2D");
    back.push_back({host, {d, count * sizeof(T)}});
    return d;
  }
  void finish(uint32_t flags) {
    for (auto& b : back)
      cuda_check(cudaMemcpyAsync(b.first, b.second.first, b.second.second, cudaMemcpyDeviceToHost, c->stream), "D2H");
    if (!dev || !(flags & DGX_ASYNC)) cuda_check(cudaStreamSynchronize(c->stream), "sync");
  }
};

size_t bytes_round(size_t n) { return (n + 255) & ~size_t(255); }

}  // namespace

extern "C" {

const char* dgx_last_error(void) { return g_err.c_str(); }
int dgx_abi_version(void) { return DGX_ABI_VERSION; }

int dgx_ctx_create(int device, dgx_ctx** out) {
  return guarded([&] {
    if (!out) throw DgxError(DGX_E_INVALID, "out is NULL");
    auto* c = new dgx_ctx();
    c->device = device;
    try {
      set_device(c);
      cudaDeviceProp prop;
      cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
      if (prop.major < 10) throw DgxError(DGX_E_UNSUPPORTED, std::string("sm_100a device required, got ") + prop.name);
      c->num_sms = prop.multiProcessorCount;
      cuda_check(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking), "cudaStreamCreate");
      c->stream = c->own;
      cuda_check(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming), "cudaEventCreate");
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

int dgx_ctx_destroy(dgx_ctx* c) {
  return guarded([&] {
    if (!c) return;
    cudaSetDevice(c->device);
    c->scratch.release();
    c->io.release();
    for (auto& sub : c->subs) {
      sub.scratch.release();
      if (sub.done) cudaEventDestroy(sub.done);
      if (sub.stream) cudaStreamDestroy(sub.stream);
    }
    for (auto& t : c->timed) {
      cudaEventDestroy(t.second.first);
      cudaEventDestroy(t.second.second);
    }
    for (auto e : c->event_pool) cudaEventDestroy(e);
    if (c->fork) cudaEventDestroy(c->fork);
    if (c->own) cudaStreamDestroy(c->own);
    delete c;
  });
}

int dgx_ctx_set_stream(dgx_ctx* c, void* s) {
  return guarded([&] {
    if (!c) throw DgxError(DGX_E_INVALID, "NULL context");
    cudaStream_t next = s ? static_cast<cudaStream_t>(s) : c->own;
    if (next != c->stream) {
      // the context's scratch (logs, ticket counter, staging) is reused by the
      // next launch: order it after everything already queued on the old stream
      set_device(c);
      cuda_check(cudaEventRecord(c->fork, c->stream), "cudaEventRecord");
      cuda_check(cudaStreamWaitEvent(next, c->fork, 0), "cudaStreamWaitEvent");
    }
    c->stream = next;
  });
}

int dgx_ctx_set_correction_capacity(dgx_ctx* c, int32_t cap) {
  return guarded([&] {
    if (cap < 1) throw DgxError(DGX_E_INVALID, "capacity must be >= 1");
    c->cap_corr = cap;
  });
}

int64_t dgx_ctx_launch_count(const dgx_ctx* c) { return c ? c->launches : 0; }

int dgx_ctx_set_adjoint(dgx_ctx* c, int variant) {
  return guarded([&] {
    if (!c) throw DgxError(DGX_E_INVALID, "NULL context");
    if (variant != DGX_ADJOINT_AUTO && variant != DGX_ADJOINT_CTA && variant != DGX_ADJOINT_LANE)
      throw DgxError(DGX_E_INVALID, "unknown adjoint variant");
    c->adjoint = variant;
  });
}

int dgx_ctx_set_kernel_timing(dgx_ctx* c, int enable) {
  return guarded([&] {
    if (!c) throw DgxError(DGX_E_INVALID, "NULL context");
    set_device(c);
    for (auto& t : c->timed) {
      c->event_pool.push_back(t.second.first);
      c->event_pool.push_back(t.second.second);
    }
    c->timed.clear();
    c->timing = enable != 0;
  });
}

int dgx_ctx_kernel_times(dgx_ctx* c, double ms[3], int64_t count[3]) {
  return guarded([&] {
    if (!c) throw DgxError(DGX_E_INVALID, "NULL context");
    set_device(c);
    double acc[3] = {0.0, 0.0, 0.0};
    int64_t n[3] = {0, 0, 0};
    for (auto& t : c->timed) {
      cuda_check(cudaEventSynchronize(t.second.second), "cudaEventSynchronize");
      float e = 0.0f;
      cuda_check(cudaEventElapsedTime(&e, t.second.first, t.second.second), "cudaEventElapsedTime");
      acc[t.first] += e;
      ++n[t.first];
    }
    for (int k = 0; k < 3; ++k) {
      if (ms) ms[k] = acc[k];
      if (count) count[k] = n[k];
    }
  });
}

int dgx_hand_upload(dgx_ctx* c, const dgx_hand_desc* d, dgx_hand** out) {
  return guarded([&] {
    if (!c || !d || !out) throw DgxError(DGX_E_INVALID, "NULL argument");
    const int L = d->num_links, J = d->num_joints, N = d->num_samples;
    if (L < 1 || J < 0 || N < 1) throw DgxError(DGX_E_INVALID, "hand: empty descriptor");
    if (J + 6 > kMaxDim) throw DgxError(DGX_E_UNSUPPORTED, "hand: more than 26 joints");
    if (L != J + 1) throw DgxError(DGX_E_INVALID, "hand: expected one parent joint per non-base link");
    // validation mirrors hand.cpp:149-210
    std::vector<int> seen(L, 0);
    for (int k = 0; k < L; ++k) {
      int li = d->topo[k];
      if (li < 0 || li >= L || seen[li]) throw DgxError(DGX_E_INVALID, "hand: topo is not a permutation");
      seen[li] = 1;
      int pj = d->link_parent_joint[li];
      if (k == 0 && pj >= 0) throw DgxError(DGX_E_INVALID, "hand: topo[0] must be the base link");
      if (k > 0) {
        if (pj < 0 || pj >= J) throw DgxError(DGX_E_INVALID, "hand: multiple base links");
        if (d->joint_child[pj] != li) throw DgxError(DGX_E_INVALID, "hand: joint child mismatch");
        int par = d->joint_parent[pj];
        bool before = false;
        for (int t = 0; t < k; ++t) before |= d->topo[t] == par;
        if (!before) throw DgxError(DGX_E_INVALID, "hand: topo order must list parents before children");
      }
    }
    for (int j = 0; j < J; ++j)
      if (!(d->lower[j] < d->upper[j])) throw DgxError(DGX_E_INVALID, "hand: joint has lower >= upper limit");
    for (int i = 0; i < N; ++i)
      if (d->sample_link[i] < 0 || d->sample_link[i] >= L) throw DgxError(DGX_E_INVALID, "hand: bad sample_link");
    auto* h = new dgx_hand();
    h->ctx = c;
    h->L = L; h->J = J; h->N = N;
    h->lower.assign(d->lower, d->lower + J);
    h->upper.assign(d->upper, d->upper + J);
    size_t ints = 2 * bytes_round(4 * L) + 2 * bytes_round(4 * std::max(J, 1)) + bytes_round(4 * N);
    size_t dbls = 2 * bytes_round(8 * 3 * std::max(J, 1)) + bytes_round(8 * 9 * std::max(J, 1)) +
                  2 * bytes_round(8 * std::max(J, 1)) + bytes_round(8 * 3 * N);
    try {
      set_device(c);
      h->mem.ensure(ints + dbls);
      char* base = static_cast<char*>(h->mem.p);
      size_t off = 0;
      auto put = [&](const void* src, size_t bytes) {
        void* dst = base + off;
        if (bytes) cuda_check(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice), "hand upload");
        off += bytes_round(std::max<size_t>(bytes, 1));
        return dst;
      };
      KHand& k = h->k;
      k.L = L; k.J = J; k.N = N;
      k.topo = static_cast<const int*>(put(d->topo, 4 * L));
      k.link_parent_joint = static_cast<const int*>(put(d->link_parent_joint, 4 * L));
      k.joint_parent = static_cast<const int*>(put(d->joint_parent, 4 * J));
      k.joint_child = static_cast<const int*>(put(d->joint_child, 4 * J));
      k.sample_link = static_cast<const int*>(put(d->sample_link, 4 * N));
      k.axis = static_cast<const double*>(put(d->axis, 8 * 3 * J));
      k.origin_t = static_cast<const double*>(put(d->origin_t, 8 * 3 * J));
      k.origin_R = static_cast<const double*>(put(d->origin_R, 8 * 9 * J));
      k.lower = static_cast<const double*>(put(d->lower, 8 * J));
      k.upper = static_cast<const double*>(put(d->upper, 8 * J));
      k.samples = static_cast<const double*>(put(d->samples, 8 * 3 * N));
    } catch (...) {
      h->mem.release();
      delete h;
      throw;
    }
    *out = h;
  });
}

int dgx_hand_free(dgx_hand* h) {
  return guarded([&] {
    if (!h) return;
    cudaSetDevice(h->ctx->device);
    h->mem.release();
    delete h;
  });
}

int dgx_object_upload(dgx_ctx* c, const dgx_object_desc* d, dgx_object** out) {
  return guarded([&] {
    if (!c || !d || !out) throw DgxError(DGX_E_INVALID, "NULL argument");
    if (!(d->mass > 0.0)) throw DgxError(DGX_E_INVALID, "object: mass must be > 0");
    auto* o = new dgx_object();
    o->ctx = c;
    o->kind = d->kind;
    try {
      set_device(c);
      o->sdf.kind = d->kind;
      if (d->kind == DGX_SDF_SPHERE) {
        if (!(d->radius > 0.0)) throw DgxError(DGX_E_INVALID, "sphere: radius must be > 0");
        o->sdf.sph = SphereSdf{V3{d->center[0], d->center[1], d->center[2]}, d->radius};
      } else if (d->kind == DGX_SDF_BOX) {
        o->sdf.box = BoxSdf{V3{d->center[0], d->center[1], d->center[2]},
                            V3{d->half_extents[0], d->half_extents[1], d->half_extents[2]}};
      } else if (d->kind == DGX_SDF_GRID) {
        if (d->dims[0] < 2 || d->dims[1] < 2 || d->dims[2] < 2 || !d->values)
          throw DgxError(DGX_E_INVALID, "grid: dims must be >= 2 and values non-NULL");
        const int nx = d->dims[0], ny = d->dims[1], nz = d->dims[2];
        const size_t n = static_cast<size_t>(nx) * ny * nz;
        const size_t nc = static_cast<size_t>(nx - 1) * (ny - 1) * (nz - 1);
        if (8 * nc >= (size_t(1) << 31) || n >= (size_t(1) << 31))
          throw DgxError(DGX_E_UNSUPPORTED, "grid: more than 2^28 cells (32-bit cell offsets)");
        // node values (host-layout copy) + the packed cells the kernels read
        // (GridSdf::cells): corner-packed (8 values per cell, one sector per
        // lookup) while that copy stays well inside L2, else xy-quads (4 per
        // cell per plane, half the footprint, two sectors per lookup).
        // DGX_GRID_LAYOUT=8|4 forces one (A/B measurements).
        const size_t vbytes = (n * sizeof(float) + 255) & ~size_t(255);
        int pairs = 8 * nc * sizeof(float) > (size_t(32) << 20) ? 1 : 0;
        if (const char* ev = std::getenv("DGX_GRID_LAYOUT")) pairs = std::atoi(ev) == 4 ? 1 : 0;
        const size_t ncp = pairs ? static_cast<size_t>(nx - 1) * (ny - 1) * nz : nc;  // packed units
        const int per = pairs ? 4 : 8;
        o->vals.ensure(vbytes + ncp * per * sizeof(float));
        cuda_check(cudaMemcpy(o->vals.p, d->values, n * sizeof(float), cudaMemcpyHostToDevice), "grid upload");
        std::vector<float> packed(ncp * per);
        const float* v = d->values;
        auto at = [&](int i, int j, int k) { return v[(static_cast<size_t>(k) * ny + j) * nx + i]; };
        for (int k = 0; k < (pairs ? nz : nz - 1); ++k)
          for (int j = 0; j < ny - 1; ++j)
            for (int i = 0; i < nx - 1; ++i) {
              float* c = packed.data() + per * ((static_cast<size_t>(k) * (ny - 1) + j) * (nx - 1) + i);
              c[0] = at(i, j, k); c[1] = at(i + 1, j, k); c[2] = at(i, j + 1, k); c[3] = at(i + 1, j + 1, k);
              if (!pairs) {
                c[4] = at(i, j, k + 1); c[5] = at(i + 1, j, k + 1); c[6] = at(i, j + 1, k + 1);
                c[7] = at(i + 1, j + 1, k + 1);
              }
            }
        float* dcells = reinterpret_cast<float*>(static_cast<char*>(o->vals.p) + vbytes);
        cuda_check(cudaMemcpy(dcells, packed.data(), packed.size() * sizeof(float), cudaMemcpyHostToDevice),
                   "grid cells upload");
        o->sdf.grd = GridSdf{nx, ny, nz, V3{d->origin[0], d->origin[1], d->origin[2]}, d->spacing, d->inv_spacing,
                             static_cast<const float*>(o->vals.p), dcells, pairs, static_cast<float>(d->origin[0]),
                             static_cast<float>(d->origin[1]), static_cast<float>(d->origin[2]),
                             static_cast<float>(d->spacing), static_cast<float>(d->inv_spacing)};
        // block lower bounds for the forward pre-filter (GridSdf::bmin): blocks of
        // 2^bs cells per axis, each the min over its nodes widened by one node
        // ~16 blocks along the largest axis (measured: 64^3 with 4-cell blocks
        // forward 1.61 -> 1.40 ms, 128^3 with 8-cell blocks 20.3 -> 17.4 ms per
        // 4096-candidate step; 8-cell blocks on 64^3 gain nothing)
        const int nmax = std::max(nx, std::max(ny, nz)) - 1;
        int bs = std::max(1, static_cast<int>(std::lround(std::log2(nmax / 16.0))));
        if (const char* ev = std::getenv("DGX_GRID_BLOCK")) bs = std::atoi(ev);  // 0: off (A/B)
        if (bs > 0) {
          const int bnx = ((nx - 2) >> bs) + 1, bny = ((ny - 2) >> bs) + 1, bnz = ((nz - 2) >> bs) + 1;
          std::vector<float> bm(static_cast<size_t>(bnx) * bny * bnz);
          for (int bk = 0; bk < bnz; ++bk)
            for (int bj = 0; bj < bny; ++bj)
              for (int bi = 0; bi < bnx; ++bi) {
                float mn = std::numeric_limits<float>::infinity();
                const int i0 = std::max(0, (bi << bs) - 1), i1 = std::min(nx - 1, ((bi + 1) << bs) + 1);
                const int j0 = std::max(0, (bj << bs) - 1), j1 = std::min(ny - 1, ((bj + 1) << bs) + 1);
                const int k0 = std::max(0, (bk << bs) - 1), k1 = std::min(nz - 1, ((bk + 1) << bs) + 1);
                for (int k = k0; k <= k1; ++k)
                  for (int j = j0; j <= j1; ++j)
                    for (int i = i0; i <= i1; ++i) mn = std::min(mn, at(i, j, k));
                bm[(static_cast<size_t>(bk) * bny + bj) * bnx + bi] = mn;
              }
          o->bmin.ensure(bm.size() * sizeof(float));
          cuda_check(cudaMemcpy(o->bmin.p, bm.data(), bm.size() * sizeof(float), cudaMemcpyHostToDevice),
                     "grid block bounds upload");
          o->sdf.grd.bmin = static_cast<const float*>(o->bmin.p);
          o->sdf.grd.bshift = bs;
          o->sdf.grd.bnx = bnx;
          o->sdf.grd.bny = bny;
        }
      } else if (d->kind == DGX_SDF_MESH) {
        // MeshSdf(TriMesh, alpha_phong) (sdf.cpp:17-20): validate, BVH, upload
        if (!(d->alpha_phong >= 0.0 && d->alpha_phong <= 1.0))
          throw std::invalid_argument("alpha_phong must be in [0,1]");
        if (d->num_faces >= (1 << 30))
          throw DgxError(DGX_E_UNSUPPORTED, "mesh: more than 2^30 faces (packed face ids)");
        MeshHost mh;
        mesh_prepare(d->num_vertices, d->vertices, d->num_faces, d->faces, d->vertex_normals, mh);
        auto rnd = [](size_t x) { return (x + 255) & ~size_t(255); };
        const size_t b_nodes = rnd(mh.nodes.size() * sizeof(MeshNode)), b_faces = rnd(mh.faces.size() * sizeof(MeshFace));
        const size_t b_tri = rnd(mh.tri.size() * sizeof(int)), b_v = rnd(mh.vx.size() * sizeof(double));
        const size_t b_vfo = rnd(mh.vf_off.size() * sizeof(int)), b_vfi = rnd(mh.vf_idx.size() * sizeof(int));
        const size_t total = b_nodes + b_faces + b_tri + 2 * b_v + b_vfo + b_vfi + rnd(sizeof(MeshGeom));
        o->vals.ensure(total);
        char* base = static_cast<char*>(o->vals.p);
        MeshGeom g{};
        size_t off = 0;
        auto put = [&](const void* src, size_t bytes, size_t span) {
          cuda_check(cudaMemcpy(base + off, src, bytes, cudaMemcpyHostToDevice), "mesh upload");
          void* dst = base + off;
          off += span;
          return dst;
        };
        g.nodes = static_cast<const MeshNode*>(put(mh.nodes.data(), mh.nodes.size() * sizeof(MeshNode), b_nodes));
        g.faces = static_cast<const MeshFace*>(put(mh.faces.data(), mh.faces.size() * sizeof(MeshFace), b_faces));
        g.tri = static_cast<const int*>(put(mh.tri.data(), mh.tri.size() * sizeof(int), b_tri));
        g.vx = static_cast<const double*>(put(mh.vx.data(), mh.vx.size() * sizeof(double), b_v));
        g.vn = static_cast<const double*>(put(mh.vn.data(), mh.vn.size() * sizeof(double), b_v));
        g.vf_off = static_cast<const int*>(put(mh.vf_off.data(), mh.vf_off.size() * sizeof(int), b_vfo));
        g.vf_idx = static_cast<const int*>(put(mh.vf_idx.data(), mh.vf_idx.size() * sizeof(int), b_vfi));
        for (int k = 0; k < 3; ++k) {
          g.blo[k] = mh.blo[k];
          g.bhi[k] = mh.bhi[k];
        }
        g.alpha = d->alpha_phong;
        mesh_ray_dirs(g.dir, g.inv);
        g.cull = 0.005;  // ContactSolver::kCullMargin (sim.hpp:213)
        g.nfaces = d->num_faces;
        o->sdf.mesh = MeshSdf{static_cast<const MeshGeom*>(put(&g, sizeof(MeshGeom), rnd(sizeof(MeshGeom))))};
        o->mesh_vx = g.vx;
        o->mesh_nv = d->num_vertices;
      } else {
        throw DgxError(DGX_E_UNSUPPORTED, "object: unknown SDF kind " + std::to_string(d->kind));
      }
      o->k.mass = d->mass;
      o->k.inv_mass = 1.0 / d->mass;
      o->k.com = V3{d->com[0], d->com[1], d->com[2]};
      for (int t = 0; t < 9; ++t) o->k.inertia_body_inv.m[t] = d->inertia_body_inv[t];
      for (int t = 0; t < 9; ++t) {
        o->inertia_body.m[t] = d->inertia_body[t];
        o->has_inertia_body = o->has_inertia_body || d->inertia_body[t] != 0.0;
      }
      // predict() from the canonical state (thetadot = 0, sim.hpp:74-83) and
      // world_inertia_inv (sim.hpp:96-100), same formulas as the kernel
      const Q4 pred_q = qnormalized(qmul(quat_exp(V3{0.0, 0.0, 0.0}), Q4{1.0, 0.0, 0.0, 0.0}));
      const M3 Rp = rotation_matrix(pred_q);
      o->k.Iw = mul(mul(Rp, o->k.inertia_body_inv), transposed(Rp));
    } catch (...) {
      o->vals.release();
      o->bmin.release();
      delete o;
      throw;
    }
    *out = o;
  });
}

int dgx_object_free(dgx_object* o) {
  return guarded([&] {
    if (!o) return;
    cudaSetDevice(o->ctx->device);
    o->vals.release();
    o->bmin.release();
    delete o;
  });
}

int dgx_sdf_query_batch(dgx_ctx* c, const dgx_object* o, int32_t n, const double* points, double radius,
                        int32_t within, double* out, uint32_t flags) {
  return guarded([&] {
    if (!c || !o) throw DgxError(DGX_E_INVALID, "NULL argument");
    if (n < 0) throw DgxError(DGX_E_INVALID, "n < 0");
    if (radius < 0.0) throw std::invalid_argument("dilation radius must be >= 0");
    if (n == 0) return;
    set_device(c);
    const bool dev = flags & DGX_DEVICE_PTRS;
    Staging s(c, dev, bytes_round(24ull * n) + bytes_round(64ull * n));
    const double* dp = s.in(points, static_cast<size_t>(n) * 3);
    double* dq = s.out(out, static_cast<size_t>(n) * 8);
    cuda_check(launch_sdf_query(o->sdf, n, dp, radius, within, dq, c->stream), "sdf_query_kernel");
    ++c->launches;
    s.finish(flags);
  });
}

int dgx_mesh_inertia(int32_t num_vertices, const double* vertices, int32_t num_faces, const int32_t* faces,
                     double density, double* mass, double* com, double* inertia, double* inertia_inv) {
  return guarded([&] {
    if (!mass || !com || !inertia || !inertia_inv) throw DgxError(DGX_E_INVALID, "NULL argument");
    mesh_inertia(num_vertices, vertices, num_faces, faces, density, *mass, com, inertia, inertia_inv);
  });
}

int dgx_mesh_bvh(int32_t num_vertices, const double* vertices, int32_t num_faces, const int32_t* faces, int32_t cap,
                 double* boxes, int32_t* links, int32_t* face_order, int32_t* n_nodes) {
  return guarded([&] {
    if (!boxes || !links || !face_order || !n_nodes) throw DgxError(DGX_E_INVALID, "NULL argument");
    MeshHost mh;
    mesh_prepare(num_vertices, vertices, num_faces, faces, nullptr, mh);
    const int n = static_cast<int>(mh.nodes.size());
    if (n > cap) throw DgxError(DGX_E_INVALID, "cap < node count " + std::to_string(n));
    for (int i = 0; i < n; ++i) {
      const MeshNode& nd = mh.nodes[i];
      for (int k = 0; k < 3; ++k) {
        boxes[6 * i + k] = nd.lo[k];
        boxes[6 * i + 3 + k] = nd.hi[k];
      }
      links[4 * i] = nd.left; links[4 * i + 1] = nd.right; links[4 * i + 2] = nd.first; links[4 * i + 3] = nd.count;
    }
    for (int i = 0; i < num_faces; ++i) face_order[i] = mh.faces[i].f;
    *n_nodes = n;
  });
}

int dgx_contacts_batch(dgx_ctx* c, const dgx_hand* h, const dgx_object* o, int32_t B, const double* q,
                       const double* sample_area, int32_t T, const double* thresholds, int32_t cap,
                       double* contact_area, int32_t* contact_count, int32_t* num_contacts, int32_t* contact_index,
                       double* contacts, uint32_t flags) {
  return guarded([&] {
    if (!c || !h || !o || !sample_area || !thresholds || !contact_area || !contact_count || !num_contacts)
      throw DgxError(DGX_E_INVALID, "NULL argument");
    if (B < 0 || cap < 0) throw DgxError(DGX_E_INVALID, "B < 0 or cap < 0");
    if (T < 1 || T > 16) throw DgxError(DGX_E_INVALID, "contacts: 1..16 thresholds");
    for (int t = 0; t < T; ++t)
      if (!(thresholds[t] >= 0.0) || (t > 0 && thresholds[t] < thresholds[t - 1]))
        throw std::invalid_argument("contacts: thresholds must be >= 0 and ascending");
    if (cap > 0 && (!contact_index || !contacts)) throw DgxError(DGX_E_INVALID, "contacts: cap > 0 needs outputs");
    if (B == 0) return;
    set_device(c);
    const bool dev = flags & DGX_DEVICE_PTRS;
    const size_t N = h->N;
    Staging s(c, dev, bytes_round(8ull * B * (7 + h->J)) + bytes_round(8ull * N) + bytes_round(8ull * B * T) +
                          bytes_round(4ull * B * T) + bytes_round(4ull * B) + bytes_round(4ull * B * cap) +
                          bytes_round(56ull * B * cap));
    const double* dq = s.in(q, static_cast<size_t>(B) * (7 + h->J));
    const double* da = s.in(sample_area, N);
    double* dca = s.out(contact_area, static_cast<size_t>(B) * T);
    int* dcnt = s.out(contact_count, static_cast<size_t>(B) * T);
    int* dn = s.out(num_contacts, static_cast<size_t>(B));
    int* dci = s.out(contact_index, static_cast<size_t>(B) * cap);
    double* dcr = s.out(contacts, static_cast<size_t>(B) * cap * 7);
    c->scratch.thr.ensure(16 * sizeof(double));
    cuda_check(cudaMemcpyAsync(c->scratch.thr.p, thresholds, T * sizeof(double), cudaMemcpyHostToDevice, c->stream),
               "H2D thresholds");
    const int grid = std::min(B, c->num_sms * 8);
    cuda_check(launch_contacts(h->k, o->sdf, B, dq, da, T, static_cast<const double*>(c->scratch.thr.p), cap, dca,
                               dcnt, dn, dci, dcr, grid, c->stream),
               "contacts_kernel");
    ++c->launches;
    s.finish(flags);
  });
}

int dgx_drop_batch(dgx_ctx* c, const dgx_object* o, int32_t B, const double* state_in, const dgx_drop_params* p,
                   double* state_out, int32_t* steps, double* ke, double* stats, double* traj, uint32_t flags) {
  return guarded([&] {
    if (!c || !o || !p || !steps || !ke) throw DgxError(DGX_E_INVALID, "NULL argument");
    if (B < 0) throw DgxError(DGX_E_INVALID, "B < 0");
    if (o->kind != DGX_SDF_MESH || !o->mesh_vx)
      throw DgxError(DGX_E_UNSUPPORTED, "drop: needs a mesh object (its vertices are the table contacts, sim.cpp:28)");
    if (!o->has_inertia_body) throw DgxError(DGX_E_INVALID, "drop: object descriptor lacks inertia_body");
    if (!(p->dt > 0.0) || p->gs_iters < 0 || p->max_steps < 0)
      throw DgxError(DGX_E_INVALID, "drop: dt > 0, gs_iters >= 0, max_steps >= 0 required");
    if (traj && p->record_every <= 0) throw DgxError(DGX_E_INVALID, "drop: traj needs record_every > 0");
    if (p->settle_steps < 1) throw DgxError(DGX_E_INVALID, "drop: settle_steps must be >= 1");
    if (B == 0) return;
    set_device(c);
    DropObj O{o->mesh_vx, o->mesh_nv, o->k.mass, o->k.com, o->inertia_body, o->k.inertia_body_inv};
    DropParams P{p->dt, p->mu, p->gs_iters, V3{p->gravity[0], p->gravity[1], p->gravity[2]}, p->max_steps,
                 p->min_steps, p->ke_tol, p->record_every, p->settle_steps, p->measure_residual};
    const int rows = traj ? p->max_steps / p->record_every : 0;
    const bool dev = flags & DGX_DEVICE_PTRS;
    Staging s(c, dev, bytes_round(104ull * B) * 2 + bytes_round(4ull * B) + bytes_round(8ull * B) +
                          bytes_round(32ull * B) + bytes_round(104ull * B * rows));
    const double* din = s.in(state_in, static_cast<size_t>(B) * 13);
    double* dout = s.out(state_out, static_cast<size_t>(B) * 13);
    int* dsteps = s.out(steps, static_cast<size_t>(B));
    double* dke = s.out(ke, static_cast<size_t>(B));
    double* dstats = s.out(stats, static_cast<size_t>(B) * 4);
    double* dtraj = s.out(traj, static_cast<size_t>(B) * rows * 13);
    const int warps = std::min(B, c->num_sms * 32);
    c->scratch.drop.ensure(static_cast<size_t>(warps) * o->mesh_nv * sizeof(double));
    cuda_check(launch_drop(O, P, B, din, dout, dsteps, dke, dstats, static_cast<double*>(c->scratch.drop.p), warps,
                           dtraj, c->stream),
               "drop_kernel");
    ++c->launches;
    s.finish(flags);
  });
}

int dgx_forward_batch(dgx_ctx* c, const dgx_hand* h, int32_t B, const double* q, double* points, uint32_t flags) {
  return guarded([&] {
    if (B < 0) throw DgxError(DGX_E_INVALID, "B < 0");
    if (B == 0) return;
    set_device(c);
    const bool dev = flags & DGX_DEVICE_PTRS;
    Staging s(c, dev, bytes_round(8ull * B * (7 + h->J)) + bytes_round(24ull * B * h->N));
    const double* dq = s.in(q, static_cast<size_t>(B) * (7 + h->J));
    double* dp = s.out(points, static_cast<size_t>(B) * h->N * 3);
    int grid = std::min(B, c->num_sms * 4);
    cuda_check(launch_forward(h->k, dq, dp, B, grid, c->stream), "forward_kernel");
    ++c->launches;
    s.finish(flags);
  });
}

static void run_fused(dgx_ctx* c, const dgx_hand* h, const dgx_object* o, int32_t B, const double* q,
                      double* qio, double* am, double* av, KSim S, const KOpt& P, int mode, double* losses,
                      double* grads, double* stats, double* sim_res, double* sim_grads, double* point_grads,
                      double* traj, int32_t* status, uint32_t flags) {
  if (!c || !h || !o) throw DgxError(DGX_E_INVALID, "NULL handle");
  if (B < 0) throw DgxError(DGX_E_INVALID, "B < 0");
  if (B == 0) return;
  set_device(c);
  const bool dev = flags & DGX_DEVICE_PTRS;
  const int M = S.M, D = 6 + h->J, Qd = 7 + h->J, N = h->N;
  const int steps = mode == kModeOpt ? (P.k_end - P.k_begin) : 0;
  size_t total = bytes_round(8ull * B * Qd) + 2 * bytes_round(8ull * B * D) + bytes_round(8ull * B * 3) +
                 bytes_round(8ull * B * 3 * D) + bytes_round(8ull * B * M * 5) + bytes_round(8ull * B * M) +
                 bytes_round(8ull * B * M * D) + (point_grads ? bytes_round(24ull * B * M * N) : 0) +
                 (traj ? bytes_round(8ull * B * steps * (3 + D)) : 0) + bytes_round(4ull * B);
  Staging s(c, dev, total);
  KBuf buf{};
  if (mode == kModeOpt) {
    buf.q = s.out(qio, static_cast<size_t>(B) * Qd, true);
    buf.adam_m = s.out(am, static_cast<size_t>(B) * D, true);
    buf.adam_v = s.out(av, static_cast<size_t>(B) * D, true);
  } else {
    buf.q = const_cast<double*>(s.in(q, static_cast<size_t>(B) * Qd));
  }
  buf.losses = s.out(losses, static_cast<size_t>(B) * 3);
  buf.grads = s.out(grads, static_cast<size_t>(B) * 3 * D);
  buf.stats = s.out(stats, static_cast<size_t>(B) * M * 5);
  buf.sim_res = s.out(sim_res, static_cast<size_t>(B) * M);
  buf.sim_grads = s.out(sim_grads, static_cast<size_t>(B) * M * D);
  buf.point_grads = s.out(point_grads, static_cast<size_t>(B) * M * N * 3);
  buf.traj = s.out(traj, static_cast<size_t>(B) * steps * (3 + D));
  // rows of iterates after a candidate's failure are never written: zero, not stale staging
  if (buf.traj && B > 0 && steps > 0)
    cuda_check(cudaMemsetAsync(buf.traj, 0, sizeof(double) * B * steps * (3 + D), c->stream), "cudaMemsetAsync");
  if (!status) throw DgxError(DGX_E_INVALID, "status is NULL");
  buf.status = s.out(status, static_cast<size_t>(B));
  if (point_grads) cuda_check(cudaMemsetAsync(buf.point_grads, 0, 24ull * B * M * N, c->stream), "memset");
  buf.egrad = nullptr;
  launch_range(c, c->scratch, h, o, S, P, buf, B, mode, c->stream);
  s.finish(flags);
}

int dgx_loss_gradient_batch(dgx_ctx* c, const dgx_hand* h, const dgx_object* o, int32_t B, const double* q,
                            const dgx_params* p, double* losses, double* grads, int32_t* status, uint32_t flags) {
  return guarded([&] {
    KSim S = make_sim(p, false);
    upload_velocities(c, S, p);
    KOpt P{};
    run_fused(c, h, o, B, q, nullptr, nullptr, nullptr, S, P, kModeGrad, losses, grads, nullptr, nullptr, nullptr,
              nullptr, nullptr, status, flags);
  });
}

int dgx_evaluate_losses_batch(dgx_ctx* c, const dgx_hand* h, const dgx_object* o, int32_t B, const double* q,
                              const dgx_params* p, double* losses, double* stats, int32_t* status, uint32_t flags) {
  return guarded([&] {
    KSim S = make_sim(p, true);
    upload_velocities(c, S, p);
    KOpt P{};
    run_fused(c, h, o, B, q, nullptr, nullptr, nullptr, S, P, kModeEval, losses, nullptr, stats, nullptr, nullptr,
              nullptr, nullptr, status, flags);
  });
}

int dgx_debug_sims(dgx_ctx* c, const dgx_hand* h, const dgx_object* o, int32_t B, const double* q,
                   const dgx_params* p, double* sim_res, double* sim_grads, double* point_grads, int32_t* status,
                   uint32_t flags) {
  return guarded([&] {
    KSim S = make_sim(p, false);
    upload_velocities(c, S, p);
    KOpt P{};
    run_fused(c, h, o, B, q, nullptr, nullptr, nullptr, S, P, kModeGrad, nullptr, nullptr, nullptr, sim_res,
              sim_grads, point_grads, nullptr, status, flags);
  });
}

int dgx_optimize_batch(dgx_ctx* c, const dgx_hand* h, const dgx_object* o, int32_t B, double* q, double* am,
                       double* av, const dgx_params* p, const dgx_opt* opt, double* traj, int32_t* status,
                       uint32_t flags) {
  return guarded([&] {
    if (!opt) throw DgxError(DGX_E_INVALID, "opt is NULL");
    if (opt->iters < 1 || opt->k_begin < 0 || opt->k_end < opt->k_begin || opt->k_end > opt->iters)
      throw DgxError(DGX_E_INVALID, "opt: need 0 <= k_begin <= k_end <= iters, iters >= 1");
    if (!(opt->lr > 0.0)) throw DgxError(DGX_E_INVALID, "opt: learning rate must be > 0");
    KSim S = make_sim(p, false);
    upload_velocities(c, S, p);
    KOpt P{opt->iters, opt->k_begin, opt->k_end, opt->record, opt->r0, opt->lr, opt->beta1, opt->beta2, opt->eps};
    run_fused(c, h, o, B, nullptr, q, am, av, S, P, kModeOpt, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
              opt->record ? traj : nullptr, status, flags);
  });
}

int dgx_optimize_multi(dgx_ctx* c, const dgx_hand* h, int32_t n_obj, const dgx_object* const* objs,
                       const int32_t* counts, double* q, double* am, double* av, const dgx_params* p,
                       const dgx_opt* opt, double* traj, int32_t* status, uint32_t flags) {
  return guarded([&] {
    if (!c || !h || !objs || !counts || !opt || !status) throw DgxError(DGX_E_INVALID, "NULL argument");
    if (n_obj < 0) throw DgxError(DGX_E_INVALID, "n_obj < 0");
    if (opt->iters < 1 || opt->k_begin < 0 || opt->k_end < opt->k_begin || opt->k_end > opt->iters)
      throw DgxError(DGX_E_INVALID, "opt: need 0 <= k_begin <= k_end <= iters, iters >= 1");
    if (!(opt->lr > 0.0)) throw DgxError(DGX_E_INVALID, "opt: learning rate must be > 0");
    int64_t B64 = 0;
    for (int i = 0; i < n_obj; ++i) {
      if (!objs[i] || counts[i] < 0) throw DgxError(DGX_E_INVALID, "bad object / count");
      B64 += counts[i];
    }
    if (B64 == 0) return;
    if (B64 > INT32_MAX) throw DgxError(DGX_E_INVALID, "too many candidates");
    const int B = static_cast<int>(B64);
    set_device(c);
    KSim S0 = make_sim(p, false);
    upload_velocities(c, S0, p);
    KOpt P{opt->iters, opt->k_begin, opt->k_end, opt->record, opt->r0, opt->lr, opt->beta1, opt->beta2, opt->eps};
    const bool dev = flags & DGX_DEVICE_PTRS;
    const int D = 6 + h->J, Qd = 7 + h->J, steps = opt->k_end - opt->k_begin;
    Staging st(c, dev, bytes_round(8ull * B * Qd) + 2 * bytes_round(8ull * B * D) + bytes_round(4ull * B) +
                           (opt->record && traj ? bytes_round(8ull * B * steps * (3 + D)) : 0));
    double* dq = st.out(q, static_cast<size_t>(B) * Qd, true);
    double* dm = st.out(am, static_cast<size_t>(B) * D, true);
    double* dv = st.out(av, static_cast<size_t>(B) * D, true);
    double* dt = st.out(opt->record ? traj : nullptr, static_cast<size_t>(B) * steps * (3 + D));
    if (dt && B > 0 && steps > 0)  // rows after a candidate's failure stay zero
      cuda_check(cudaMemsetAsync(dt, 0, sizeof(double) * B * steps * (3 + D), c->stream), "cudaMemsetAsync");
    int32_t* ds = st.out(status, static_cast<size_t>(B));
    // fork onto the side streams (object i -> stream i % P), each with its own scratch
    int n_live = 0;
    for (int i = 0; i < n_obj; ++i) n_live += counts[i] > 0 ? 1 : 0;
    int max_streams = 4;
    if (const char* ev = std::getenv("DGX_STREAMS")) max_streams = std::max(1, std::atoi(ev));  // A/B
    const int P_streams = std::max(1, std::min<int>(n_obj, max_streams));
    const int concurrent = std::max(1, std::min(n_live, P_streams));
    while (static_cast<int>(c->subs.size()) < P_streams) {
      SubStream sub;
      cuda_check(cudaStreamCreateWithFlags(&sub.stream, cudaStreamNonBlocking), "cudaStreamCreate");
      cuda_check(cudaEventCreateWithFlags(&sub.done, cudaEventDisableTiming), "cudaEventCreate");
      c->subs.push_back(sub);
    }
    cuda_check(cudaEventRecord(c->fork, c->stream), "cudaEventRecord");
    for (int k = 0; k < P_streams; ++k) cuda_check(cudaStreamWaitEvent(c->subs[k].stream, c->fork, 0), "wait");
    size_t off = 0;
    for (int i = 0; i < n_obj; ++i) {
      const int Bi = counts[i];
      if (Bi == 0) continue;
      SubStream& sub = c->subs[i % P_streams];
      KSim S = S0;
      KBuf buf{};
      buf.q = dq + off * Qd;
      buf.adam_m = dm + off * D;
      buf.adam_v = dv + off * D;
      buf.traj = dt ? dt + off * steps * (3 + D) : nullptr;
      buf.status = ds + off;
      launch_range(c, sub.scratch, h, objs[i], S, P, buf, Bi, kModeOpt, sub.stream, concurrent);
      off += Bi;
    }
    for (int k = 0; k < P_streams; ++k) {
      cuda_check(cudaEventRecord(c->subs[k].done, c->subs[k].stream), "cudaEventRecord");
      cuda_check(cudaStreamWaitEvent(c->stream, c->subs[k].done, 0), "wait");
    }
    st.finish(flags);
  });
}

int dgx_grasp_energy_batch(dgx_ctx* c, const dgx_hand* h, const dgx_object* o, int32_t B, const double* q,
                           const dgx_params* p, double* energy, double* grads, uint32_t flags) {
  return guarded([&] {
    if (!c || !h || !o || !p || !energy) throw DgxError(DGX_E_INVALID, "NULL argument");
    if (B < 0) throw DgxError(DGX_E_INVALID, "B < 0");
    if (B == 0) return;
    set_device(c);
    KSim S{};
    S.fc_thr = p->contact_threshold > 0.0 ? p->contact_threshold : 0.005;
    S.fc_scale = p->torque_scale > 0.0 ? p->torque_scale : 0.05;
    S.w_fc = p->w_force_closure;
    S.w_pen = p->w_penetration;
    const bool dev = flags & DGX_DEVICE_PTRS;
    const int D = 6 + h->J, Qd = 7 + h->J;
    Staging s(c, dev, bytes_round(8ull * B * Qd) + bytes_round(16ull * B) + bytes_round(16ull * B * D));
    const double* dq = s.in(q, static_cast<size_t>(B) * Qd);
    double* de = s.out(energy, static_cast<size_t>(B) * 2);
    double* dg = s.out(grads, static_cast<size_t>(B) * 2 * D);
    (void)cudaGetLastError();
    cuda_check(launch_energy(h->k, o->k, o->sdf, S, B, dq, nullptr, de, dg, nullptr, std::min(B, c->num_sms * 4),
                             c->stream),
               "energy_kernel");
    ++c->launches;
    s.finish(flags);
  });
}

int dgx_apply_gradient_step_batch(dgx_ctx* c, const dgx_hand* h, int32_t B, const double* q, const double* g,
                                  double lr, double* q_out, uint32_t flags) {
  if (!h) {
    g_err = "NULL hand";
    return DGX_E_INVALID;
  }
  return dgx_apply_gradient_step_joints(c, h->J, B, q, g, lr, q_out, flags);
}

int dgx_apply_gradient_step_joints(dgx_ctx* c, int32_t J, int32_t B, const double* q, const double* g, double lr,
                                   double* q_out, uint32_t flags) {
  return guarded([&] {
    if (!c) throw DgxError(DGX_E_INVALID, "NULL context");
    if (J < 0 || J + 6 > kMaxDim) throw DgxError(DGX_E_INVALID, "num_joints out of range");
    if (B <= 0) return;
    set_device(c);
    const bool dev = flags & DGX_DEVICE_PTRS;
    const int Qd = 7 + J, D = 6 + J;
    Staging s(c, dev, 2 * bytes_round(8ull * B * Qd) + bytes_round(8ull * B * D));
    const double* dq = s.in(q, static_cast<size_t>(B) * Qd);
    const double* dg = s.in(g, static_cast<size_t>(B) * D);
    double* dout = s.out(q_out, static_cast<size_t>(B) * Qd);
    cuda_check(launch_step(J, dq, dg, lr, dout, B, c->stream), "step_kernel");
    ++c->launches;
    s.finish(flags);
  });
}

}  // extern "C"
