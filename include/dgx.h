/*
 * dgx.h — C ABI of the B200-native batched grasp search (libdgx_cuda.so).
 *
 * Plain pointers and sizes only; no CUDA / C++ / torch types in signatures.
 * Every entry point replaces one reference C++ interface of the hot path
 * (/root/reference/proj/include/diffgrasp), batched over B candidates:
 *
 *   dgx_hand_upload            dg::HandModel (hand.hpp:53-102): descriptor of a
 *                              loaded / assembled hand (samples in forward()
 *                              order, hand.hpp:143-151)
 *   dgx_object_upload          dg::GraspObject (losses.hpp:38-44): SDF backend
 *                              (incl. dg::MeshSdf over a TriMesh, sdf.hpp:21-53)
 *                              + InertialData (rigid.hpp:8-13)
 *   dgx_sdf_query_batch        MeshSdf::dilated / dilated_within (sdf.hpp:41-45)
 *   dgx_mesh_inertia           dg::inertia_from_mesh (rigid.cpp:24-94)
 *   dgx_contacts_batch         SPEC metrics.generate_contacts / contact_area
 *                              (not implemented by the reference)
 *   dgx_drop_batch             dg::step_on_table (sim.cpp:14-94) + kinetic_energy
 *                              (sim.cpp:8-12), iterated per scene
 *   dgx_forward_batch          HandModel::forward(const HandConfig&) (hand.hpp:86)
 *   dgx_loss_gradient_batch    dg::loss_gradient (losses.hpp:126-127, losses.cpp:20-66)
 *   dgx_evaluate_losses_batch  dg::evaluate_losses (losses.hpp:119-121, losses.cpp:7-18)
 *                              + SolveStats (sim.hpp:42-49) per perturbation
 *   dgx_apply_gradient_step_batch  dg::apply_gradient_step (losses.hpp:136, losses.cpp:92-102)
 *   dgx_grasp_energy_batch     north_star (3) force-closure + penetration terms
 *                              (no reference counterpart; parity-unpinned, off by default)
 *   dgx_optimize_batch         the synthesis loop the reference specifies but does
 *                              not implement:
 *                              linear dilation schedule + loss_gradient + Adam +
 *                              apply_gradient_step, fused in one launch
 *
 * Layouts (row-major, double unless noted):
 *   q      [B, 7+J]  base position (3) | base quaternion w,x,y,z (4) | joints (J)
 *                    (dg::HandConfig, hand.hpp:15-19)
 *   grads  [B, 3, 6+J]  d_stable | d_qrange | d_qlimit, each in the reference's
 *                    gradient layout [pos 3 | orientation tangent 3 | joints J]
 *                    (dg::LossGradient, losses.hpp:104-116)
 *   losses [B, 3]    stable, qrange, qlimit (dg::LossBreakdown, losses.hpp:95-102)
 *
 * Errors: functions return DGX_OK or an error code; dgx_last_error() gives the
 * thread-local message. Per-candidate failures (the reference throws
 * std::runtime_error for that candidate, losses.cpp:15-16, tape.cpp:35-38) are
 * reported in status[b] and do not affect other candidates.
 * Calls are synchronous on the context's stream unless DGX_ASYNC is given.
 */
#ifndef DGX_H_
#define DGX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DGX_ABI_VERSION 2

typedef struct dgx_ctx dgx_ctx;
typedef struct dgx_hand dgx_hand;
typedef struct dgx_object dgx_object;

/* return / per-candidate status codes */
enum {
  DGX_OK = 0,
  DGX_E_NONFINITE_LOSS = 1,  /* "loss evaluation produced a non-finite value" (losses.cpp:15-16) */
  DGX_E_NONFINITE_GRAD = 2,  /* "tape: non-finite adjoint" (tape.cpp:35-38) */
  DGX_E_CORR_OVERFLOW = 3,   /* more active corrections than the context's log capacity */
  DGX_E_SLOT_OVERFLOW = 4,   /* reserved (contact slots are sized N, as sim.hpp:155) */
  DGX_E_REPLAY = 5,          /* internal: adjoint replay disagreed with the forward */
  DGX_E_INVALID = 100,       /* invalid argument (std::invalid_argument / runtime_error) */
  DGX_E_CUDA = 101,
  DGX_E_UNSUPPORTED = 102
};

/* flags */
#define DGX_DEVICE_PTRS 1u  /* array arguments are device pointers on the context's device */
#define DGX_ASYNC 2u        /* do not synchronize the stream before returning (device ptrs only) */

typedef struct {
  int32_t num_links, num_joints, num_samples;
  const int32_t* topo;               /* [L] BFS order, parent before child (hand.hpp:97) */
  const int32_t* link_parent_joint;  /* [L] -1 for the base link (hand.hpp:47) */
  const int32_t* joint_parent;       /* [J] (hand.hpp:31) */
  const int32_t* joint_child;        /* [J] (hand.hpp:32) */
  const double* axis;                /* [J,3] unit, child origin frame (hand.hpp:33) */
  const double* origin_R;            /* [J,9] row-major (hand.hpp:34) */
  const double* origin_t;            /* [J,3] (hand.hpp:35) */
  const double* lower;               /* [J] (hand.hpp:36) */
  const double* upper;               /* [J] (hand.hpp:37) */
  const double* samples;             /* [N,3] link-frame samples in forward() order */
  const int32_t* sample_link;        /* [N] (hand.hpp:76) */
} dgx_hand_desc;

enum { DGX_SDF_SPHERE = 1, DGX_SDF_BOX = 2, DGX_SDF_GRID = 4, DGX_SDF_MESH = 8 };

typedef struct {
  int32_t kind;
  double center[3];        /* sphere / box */
  double radius;           /* sphere */
  double half_extents[3];  /* box */
  int32_t dims[3];         /* grid nx, ny, nz (x fastest) */
  double origin[3];        /* grid node (0,0,0) */
  double spacing;          /* grid node spacing h */
  double inv_spacing;      /* 1/h as used by the query (pass exactly what the oracle uses) */
  const float* values;     /* grid [nz][ny][nx]; host memory (copied) */
  double mass;             /* InertialData (rigid.hpp:8-13) */
  double com[3];
  double inertia_body_inv[9];
  /* mesh (DGX_SDF_MESH): dg::TriMesh (mesh.hpp:15-21) + MeshSdf alpha_phong
     (sdf.hpp:24). Validated as TriMesh::finalize (mesh.cpp:12-71); host memory
     (copied). The BVH is built as Bvh::build (bvh.cpp:148-163). */
  int32_t num_vertices, num_faces;
  const double* vertices;        /* [V,3] */
  const int32_t* faces;          /* [F,3] outward (counter-clockwise) winding */
  const double* vertex_normals;  /* [V,3] unit (TriMesh::set_vertex_normals), or NULL:
                                    area-weighted face normals (mesh.cpp:60-70) */
  double alpha_phong;            /* in [0,1] (sdf.cpp:19) */
  double inertia_body[9];        /* InertialData::inertia_body (rigid.hpp:11); needed by
                                    dgx_drop_batch (kinetic_energy, sim.cpp:8-12) only */
} dgx_object_desc;

/* scene drop (step_on_table, sim.cpp:14-94, iterated by a driver) */
typedef struct {
  double dt;               /* SimParams::dt */
  double mu;               /* SimParams::mu */
  int32_t gs_iters;        /* SimParams::gs_iters */
  int32_t measure_residual;/* SolveStats::measure_residual: max table penetration */
  double gravity[3];       /* SimParams::gravity (e.g. 0, 0, -9.81) */
  int32_t max_steps;       /* step cap */
  int32_t min_steps;       /* never stop before this many steps */
  double ke_tol;           /* at rest: settle_steps consecutive contact steps with
                              kinetic_energy < ke_tol (J) */
  int32_t record_every;    /* > 0 with traj: state after every record_every-th step */
  int32_t settle_steps;    /* >= 1 */
} dgx_drop_params;

typedef struct {
  double dt;               /* SimParams::dt (sim.hpp:34) */
  double mu;               /* SimParams::mu (sim.hpp:35) */
  int32_t gs_iters;        /* SimParams::gs_iters (sim.hpp:36) */
  int32_t steps;           /* StabilityProtocol::steps (losses.hpp:18): T >= 1 steps per perturbation sim */
  double dilation_radius;  /* SimParams::dilation_radius (sim.hpp:38) */
  double alpha_leak;       /* LeakPolicy::alpha_leak (sim.hpp:23) */
  int32_t num_velocities;  /* StabilityProtocol::velocities.size() = M >= 1 (losses.hpp:17) */
  int32_t pad;
  double velocities[8][3]; /* the first min(M, 8) velocities, used when velocity_list is NULL (M <= 8) */
  double w_stable, w_qrange, w_qlimit;  /* LossWeights (losses.hpp:31-35) */
  /* ---- ABI 2 ---- */
  const double* velocity_list;  /* [M,3] host memory, any M >= 1 (copied per call); NULL: velocities[] */
  /* Grasp-energy terms of north_star (3), no reference counterpart (parity-unpinned;
     dgx_grasp_energy_batch). 0 = off: the optimizer is then bit-identical to ABI 1. */
  double w_force_closure;  /* weight of E_fc = |sum_c n_c|^2 + |sum_c (p_c - com) x n_c|^2 / l^2 */
  double w_penetration;    /* weight of E_pen = sum_i max(0, -rho_i) */
  double contact_threshold;/* sample i is a contact c when |rho_i| <= threshold (m); default 0.005 */
  double torque_scale;     /* l (m) in E_fc; default 0.05 */
} dgx_params;

typedef struct {
  int32_t iters;           /* K: schedule length; r_k = r0 (1 - k/(K-1)) */
  int32_t k_begin, k_end;  /* iterations [k_begin, k_end) run by this call */
  int32_t record;          /* nonzero: write per-iterate losses + weighted grad to traj */
  double r0, lr, beta1, beta2, eps;
} dgx_opt;

const char* dgx_last_error(void);
int dgx_abi_version(void);

int dgx_ctx_create(int device, dgx_ctx** out);
int dgx_ctx_destroy(dgx_ctx* ctx);
/* use an external cudaStream_t (NULL = the context's own stream). Work already queued on
   the previous stream is ordered before the next launch (the context scratch is reused). */
int dgx_ctx_set_stream(dgx_ctx* ctx, void* cuda_stream);
/* capacity of the per-perturbation active-correction log (default 1024) */
int dgx_ctx_set_correction_capacity(dgx_ctx* ctx, int32_t cap);
/* number of kernels this context has launched */
int64_t dgx_ctx_launch_count(const dgx_ctx* ctx);
/* Per-kernel timing (measurement only; no reference counterpart): while
 * enabled, every grasp-search launch is bracketed by CUDA events on the stream
 * it runs on. dgx_ctx_kernel_times synchronizes and returns, per kernel kind
 * (0 fused, 1 split forward, 2 split adjoint), the summed milliseconds and the
 * launch count since the last enable; ms / count may be NULL. */
int dgx_ctx_set_kernel_timing(dgx_ctx* ctx, int enable);
/* Split-execution adjoint kernel (measurement / testing; no reference
 * counterpart). DGX_ADJOINT_AUTO (default): the lane adjoint (one thread per
 * (candidate, sim)) when the batch gives it >= 3 warps per SM, else the CTA
 * adjoint (one CTA per candidate, bit-identical to the fused kernel).
 * Gradients of the two agree to rounding. The DGX_ADJ
 * environment variable (lane | cta | task) overrides AUTO. */
enum { DGX_ADJOINT_AUTO = 0, DGX_ADJOINT_CTA = 1, DGX_ADJOINT_LANE = 2 };
int dgx_ctx_set_adjoint(dgx_ctx* ctx, int variant);
int dgx_ctx_kernel_times(dgx_ctx* ctx, double ms[3], int64_t count[3]);

int dgx_hand_upload(dgx_ctx* ctx, const dgx_hand_desc* desc, dgx_hand** out);
int dgx_hand_free(dgx_hand* hand);
int dgx_object_upload(dgx_ctx* ctx, const dgx_object_desc* desc, dgx_object** out);
int dgx_object_free(dgx_object* obj);

/* SDF queries in the object's canonical frame: out [n, 8] = rho - radius,
   unit gradient (3), smoothed / proxy point (3), sign, as MeshSdf::dilated
   (sdf.hpp:41, sdf.cpp:62-67). within != 0: MeshSdf::dilated_within with the
   solver's 5 mm cull (sdf.cpp:69-81, sim.hpp:213); a culled point (nullopt)
   reports rho = +inf and sign 0. Non-mesh backends never cull. */
int dgx_sdf_query_batch(dgx_ctx* ctx, const dgx_object* obj, int32_t n, const double* points, double radius,
                        int32_t within, double* out, uint32_t flags);

/* dg::inertia_from_mesh (rigid.cpp:24-94): mass, com [3], inertia_body [9]
   and its closed-form inverse [9] (row-major) of a closed mesh at `density`. */
int dgx_mesh_inertia(int32_t num_vertices, const double* vertices, int32_t num_faces, const int32_t* faces,
                     double density, double* mass, double* com, double* inertia, double* inertia_inv);

/* Host-only inspection of the mesh BVH dgx_object_upload builds (Bvh::build,
   bvh.cpp:148-163): node boxes [n,6] (lo, hi), (left, right, first, count)
   [n,4], leaf-order face ids [F]; *n_nodes = node count (arrays sized cap). */
int dgx_mesh_bvh(int32_t num_vertices, const double* vertices, int32_t num_faces, const int32_t* faces, int32_t cap,
                 double* boxes, int32_t* links, int32_t* face_order, int32_t* n_nodes);

/* points [B, N, 3] = HandModel::forward(q_b) */
int dgx_forward_batch(dgx_ctx* ctx, const dgx_hand* hand, int32_t B, const double* q, double* points,
                      uint32_t flags);

/* losses [B,3], grads [B,3,6+J] as dg::loss_gradient */
int dgx_loss_gradient_batch(dgx_ctx* ctx, const dgx_hand* hand, const dgx_object* obj, int32_t B,
                            const double* q, const dgx_params* params, double* losses, double* grads,
                            int32_t* status, uint32_t flags);

/* losses [B,3] as dg::evaluate_losses; stats [B,M,5] (active_contacts,
   corrections, singular_skipped, max_penetration, max_friction_ratio) with
   measure_residual; stats may be NULL */
int dgx_evaluate_losses_batch(dgx_ctx* ctx, const dgx_hand* hand, const dgx_object* obj, int32_t B,
                              const double* q, const dgx_params* params, double* losses, double* stats,
                              int32_t* status, uint32_t flags);

/* q_out [B,7+J] = apply_gradient_step(q_b, g_b, lr), g [B,6+J] */
int dgx_apply_gradient_step_batch(dgx_ctx* ctx, const dgx_hand* hand, int32_t B, const double* q,
                                  const double* g, double lr, double* q_out, uint32_t flags);

/* the same without a hand handle (dg::apply_gradient_step takes no hand,
   losses.hpp:136): num_joints = J of the configurations */
int dgx_apply_gradient_step_joints(dgx_ctx* ctx, int32_t num_joints, int32_t B, const double* q, const double* g,
                                   double lr, double* q_out, uint32_t flags);

/* Fused synthesis loop: q [B,7+J], adam_m / adam_v [B,6+J] updated in place;
   traj [B, k_end-k_begin, 3+6+J] (losses, weighted gradient) when opt->record;
   rows of iterates after a candidate's failure are zero. */
int dgx_optimize_batch(dgx_ctx* ctx, const dgx_hand* hand, const dgx_object* obj, int32_t B, double* q,
                       double* adam_m, double* adam_v, const dgx_params* params, const dgx_opt* opt,
                       double* traj, int32_t* status, uint32_t flags);

/* Multi-object batch (BASELINE configs 2/4/5): candidates are object-major,
   counts[i] of them for objs[i] (q / adam / traj / status rows in that order).
   Objects are launched concurrently on context-owned side streams (each with
   its own scratch), forked from and joined back to the context stream. */
int dgx_optimize_multi(dgx_ctx* ctx, const dgx_hand* hand, int32_t n_obj, const dgx_object* const* objs,
                       const int32_t* counts, double* q, double* adam_m, double* adam_v, const dgx_params* params,
                       const dgx_opt* opt, double* traj, int32_t* status, uint32_t flags);

/* Grasp-energy terms (north_star (3): force closure + penetration; the
   reference objective has neither, so they are parity-unpinned and off by
   default). At the object's canonical pose (object frame = world), per
   candidate over every hand sample p_i (HandModel::forward order) with SDF
   value rho_i and unit gradient n_i (MeshSdf::dilated at radius 0, sdf.cpp:62-67):
     contacts C = { i : |rho_i| <= contact_threshold },
     E_fc  = |sum_{i in C} n_i|^2 + |sum_{i in C} (p_i - com) x n_i|^2 / torque_scale^2
             (the differentiable force-closure estimate of Liu et al. 2021 with unit
             contact forces along the normals),
     E_pen = sum_i max(0, -rho_i).
   Gradients hold the contact set and the normals frozen (the reference's
   frozen-coefficient convention, sim.hpp:102-104): dE_fc/dp_i = 2 (n_i x tau) / l^2
   for i in C, dE_pen/dp_i = -n_i for rho_i < 0, mapped to [pos 3 | tangent 3 |
   joints J] by the FK adjoint. energy [B,2] (E_fc, E_pen), grads [B,2,6+J]
   (may be NULL). Reads contact_threshold / torque_scale from params. The
   optimizer adds w_force_closure dE_fc + w_penetration dE_pen to its weighted
   gradient every iterate when either weight is nonzero. */
int dgx_grasp_energy_batch(dgx_ctx* ctx, const dgx_hand* hand, const dgx_object* obj, int32_t B, const double* q,
                           const dgx_params* params, double* energy, double* grads, uint32_t flags);

/* Parity / debug: per-perturbation residuals [B,M], gradients [B,M,6+J] and
   optionally d residual_m / d points [B,M,N,3] (pass NULL to skip). */
int dgx_debug_sims(dgx_ctx* ctx, const dgx_hand* hand, const dgx_object* obj, int32_t B, const double* q,
                   const dgx_params* params, double* sim_res, double* sim_grads, double* point_grads,
                   int32_t* status, uint32_t flags);

/* Contact generation for grasp metrics (no
   reference implementation): hand samples of q_b (forward order) queried
   against the object at its canonical pose; a sample is a contact at
   threshold t when |rho| <= t. thresholds [T] (host memory, ascending, T <=
   16, >= 0). Outputs: contact_area [B,T] (m^2, sum of sample_area [N] over
   contacts), contact_count [B,T], num_contacts [B] (at the largest
   threshold, may exceed cap), contact_index [B,cap] (sample indices, ascending)
   and contacts [B,cap,7] (rho, smoothed surface point (3), unit gradient (3))
   for the first min(num_contacts, cap) contacts. */
int dgx_contacts_batch(dgx_ctx* ctx, const dgx_hand* hand, const dgx_object* obj, int32_t B, const double* q,
                       const double* sample_area, int32_t num_thresholds, const double* thresholds, int32_t cap,
                       double* contact_area, int32_t* contact_count, int32_t* num_contacts,
                       int32_t* contact_index, double* contacts, uint32_t flags);

/* Batched scene drop: each row of state_in
   [B,13] (dg::RigidState: x(3), theta w,x,y,z (4), xdot(3), thetadot(3)) of a
   MESH object is advanced by step_on_table (sim.cpp:14-94) until settle_steps
   consecutive steps with contact leave kinetic_energy (sim.cpp:8-12) below
   ke_tol, or max_steps.
   state_out [B,13], steps [B] (steps taken), ke [B] (final kinetic energy),
   stats [B,4] (active_contacts, corrections, singular_skipped,
   max_penetration) of one SolveStats shared by all steps (may be NULL), traj
   [B, max_steps/record_every, 13] (may be NULL). */
int dgx_drop_batch(dgx_ctx* ctx, const dgx_object* obj, int32_t B, const double* state_in,
                   const dgx_drop_params* params, double* state_out, int32_t* steps, double* ke, double* stats,
                   double* traj, uint32_t flags);

/* Utility: measured FP64 FMA throughput of the device (TFLOP/s), the
   roofline denominator for the fused kernel. */
int dgx_fp64_peak(int device, double* tflops, double* ms);

#ifdef __cplusplus
}
#endif

#endif /* DGX_H_ */
