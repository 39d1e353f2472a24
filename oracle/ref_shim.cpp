// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the parity checker, never
// the product). Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load the library built from this.
//
// Wraps the UNMODIFIED reference (/root/reference/proj, compiled out of tree by
// oracle/Makefile) behind an extern "C" API for ctypes:
//  * hands: make_three_finger_hand / make_two_finger_hand / HandModel::load_xml
//    (assets.cpp:304-310, hand.cpp:70-136) and their descriptors;
//  * objects: dg::GraspObject (losses.hpp:38-44) whose SDF member is the
//    "AnySdf": it forwards to the real MeshSdf for mesh
//    objects (bit-identical to the reference) or evaluates one of the shared
//    non-mesh backends (paper_2306_08132_b200/csrc/dgx_geom.h) behind the
//    reference's record_dilated / dilated_within contract (sdf.cpp:69-107);
//  * the reference's loss_gradient / evaluate_losses / apply_gradient_step
//    (losses.cpp) compiled from the reference source with MeshSdf -> AnySdf;
//  * per-perturbation tape gradients (losses.cpp:32-42), d residual / d points,
//    the activation trace (every record_dilated call, sweep-major), forward
//    SolveStats (sim.hpp:42-49), and the shared synthesis driver (SURVEY
//    App. C: linear dilation schedule, Adam, apply_gradient_step) run on
//    std::threads (the tape is thread_local, tape.cpp:5).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "diffgrasp/assets.hpp"
#include "diffgrasp/hand.hpp"
#include "diffgrasp/sdf.hpp"
#include "diffgrasp/tape.hpp"
#include "dgx_geom.h"

namespace dg {

// Per-thread log of every SDF evaluation made by the solver, in call order.
struct SdfTrace {
  std::vector<double>* rho = nullptr;
};
static thread_local SdfTrace g_trace;

class AnySdf {
 public:
  AnySdf(TriMesh mesh, double alpha_phong)
      : mesh_sdf_(std::make_shared<MeshSdf>(std::move(mesh), alpha_phong)) {}

  const TriMesh& mesh() const { return mesh_sdf_->mesh(); }
  const MeshSdf* mesh_sdf() const { return mesh_sdf_.get(); }

  void use_mesh() { kind_ = 0; }
  void use_sphere(const dgx::SphereSdf& s) { kind_ = dgx::kSdfSphere; sphere_ = s; }
  void use_box(const dgx::BoxSdf& b) { kind_ = dgx::kSdfBox; box_ = b; }
  void use_grid(const dgx::GridSdf& g, std::vector<float> vals) {
    kind_ = dgx::kSdfGrid;
    grid_vals_ = std::move(vals);
    grid_ = g;
    grid_.vals = grid_vals_.data();
  }
  int kind() const { return kind_; }

  // backend query in PhongQuery form (sdf.hpp:11-17); flat is left empty
  PhongQuery query(const Vec3& r) const {
    if (kind_ == 0) return mesh_sdf_->phong(r);
    dgx::V3 rv{r.x, r.y, r.z};
    dgx::SdfQuery q;
    if (kind_ == dgx::kSdfSphere) q = sphere_.query(rv);
    else if (kind_ == dgx::kSdfBox) q = box_.query(rv);
    else q = grid_.query(rv);
    PhongQuery out;
    out.rho = q.rho;
    out.grad = {q.grad.x, q.grad.y, q.grad.z};
    out.smoothed_point = {q.proxy.x, q.proxy.y, q.proxy.z};
    out.sign = q.sign;
    return out;
  }

  PhongQuery dilated(const Vec3& r, double radius) const {
    if (radius < 0.0) throw std::invalid_argument("dilation radius must be >= 0");
    PhongQuery q = query(r);
    q.rho -= radius;
    return q;
  }

  // forward-only path (sim.hpp:177): the mesh backend keeps the reference's
  // BVH cull; the analytic / grid backends return the uncut query.
  std::optional<PhongQuery> dilated_within(const Vec3& r, double radius, double cull) const {
    std::optional<PhongQuery> q;
    if (kind_ == 0) q = mesh_sdf_->dilated_within(r, radius, cull);
    else q = dilated(r, radius);
    if (g_trace.rho) g_trace.rho->push_back(q ? q->rho : 1e300);
    return q;
  }

  // recorded path (sim.hpp:165): sdf.cpp:83-107 with the backend's proxy
  // point frozen (value from the recomputed distance, unit gradient emitted
  // as recorded scalars, interpolated-normal fallback below 1e-9).
  Rec record_dilated(const Vec3T<Rec>& r, double radius, Vec3T<Rec>* grad_out) const {
    if (kind_ == 0) {
      Rec v = mesh_sdf_->record_dilated(r, radius, grad_out);
      if (g_trace.rho) g_trace.rho->push_back(v.v);
      return v;
    }
    if (radius < 0.0) throw std::invalid_argument("dilation radius must be >= 0");
    PhongQuery q = query(Vec3{r.x.v, r.y.v, r.z.v});
    Rec dx = r.x - q.smoothed_point.x;
    Rec dy = r.y - q.smoothed_point.y;
    Rec dz = r.z - q.smoothed_point.z;
    Rec out;
    if (std::abs(q.rho) < 1e-9) {
      Rec proj = dx * Rec(q.grad.x) + dy * Rec(q.grad.y) + dz * Rec(q.grad.z);
      Rec rho = Rec(static_cast<double>(q.sign)) * proj;
      if (grad_out) *grad_out = {Rec(q.grad.x), Rec(q.grad.y), Rec(q.grad.z)};
      out = rho - Rec(radius);
    } else {
      Rec dist = sqrt(dx * dx + dy * dy + dz * dz);
      Rec rho = q.sign > 0 ? dist : -dist;
      if (grad_out) {
        Rec inv = Rec(static_cast<double>(q.sign)) / dist;
        *grad_out = {dx * inv, dy * inv, dz * inv};
      }
      out = rho - Rec(radius);
    }
    if (g_trace.rho) g_trace.rho->push_back(out.v);
    return out;
  }

 private:
  std::shared_ptr<MeshSdf> mesh_sdf_;
  int kind_ = 0;
  dgx::SphereSdf sphere_{};
  dgx::BoxSdf box_{};
  dgx::GridSdf grid_{};
  std::vector<float> grid_vals_;
};

}  // namespace dg

// The reference's objective and gradient, compiled from its own source with
// the SDF type swapped.
#define MeshSdf AnySdf
#include "losses.cpp"
#undef MeshSdf

using namespace dg;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  return 1;
}

struct Params {  // mirrors oracle/ref.py:Params (ctypes)
  double dt, mu;
  int gs_iters, steps;
  double dilation_radius, alpha_leak, speed;
  double w_stable, w_qrange, w_qlimit;
};

struct OptCfg {  // mirrors oracle/ref.py:OptCfg
  int iters, k_begin, k_end, pad;
  double r0, lr, beta1, beta2, eps;
};

SimParams sim_params(const Params& p) {
  SimParams s;
  s.dt = p.dt;
  s.mu = p.mu;
  s.gs_iters = p.gs_iters;
  s.dilation_radius = p.dilation_radius;
  s.leak.alpha_leak = p.alpha_leak;
  return s;
}

// custom velocity list (dgr_set_protocol; empty: StabilityProtocol::standard)
std::vector<Vec3> g_velocities;

StabilityProtocol protocol(const Params& p) {
  if (g_velocities.empty()) return StabilityProtocol::standard(p.speed, p.steps);
  StabilityProtocol s;
  s.velocities = g_velocities;
  s.steps = p.steps;
  return s;
}

HandConfig unpack_q(const HandModel& hand, const double* q) {
  HandConfig c;
  c.base_position = {q[0], q[1], q[2]};
  c.base_orientation = {q[3], q[4], q[5], q[6]};
  c.joint_angles.assign(q + 7, q + 7 + hand.num_joints());
  return c;
}

void pack_q(const HandConfig& c, double* q) {
  q[0] = c.base_position.x; q[1] = c.base_position.y; q[2] = c.base_position.z;
  q[3] = c.base_orientation.w; q[4] = c.base_orientation.x;
  q[5] = c.base_orientation.y; q[6] = c.base_orientation.z;
  for (std::size_t j = 0; j < c.joint_angles.size(); ++j) q[7 + j] = c.joint_angles[j];
}

// BFS order of hand.cpp:177-194 (HandModel keeps it private).
std::vector<int> topo_order(const HandModel& h) {
  std::vector<int> order{h.base_link()};
  for (std::size_t head = 0; head < order.size(); ++head)
    for (int ji = 0; ji < h.num_joints(); ++ji)
      if (h.joints()[ji].parent_link == order[head]) order.push_back(h.joints()[ji].child_link);
  return order;
}

// one recorded perturbation sim exactly as losses.cpp:32-42
Rec recorded_residual(const GraspObject& obj, const HandModel& hand, const HandConfig& q,
                      const StabilityProtocol& proto, const SimParams& sim, int m, Tape& tape,
                      std::vector<Vec3T<Rec>>* points_out) {
  PoseVars<Rec> vars = record_pose_vars(tape, q);
  std::vector<Vec3T<Rec>> points = hand.forward(vars);
  if (points_out) *points_out = points;
  return perturbation_residual(obj, points, proto.velocities[m], proto, sim);
}

}  // namespace

extern "C" {

const char* dgr_last_error() { return g_err.c_str(); }

// M velocities [M,3] for every following call (M = 0: back to standard(speed))
void dgr_set_protocol(int M, const double* v) {
  g_velocities.clear();
  for (int m = 0; m < M; ++m) g_velocities.push_back({v[3 * m], v[3 * m + 1], v[3 * m + 2]});
}

// ---- hands --------------------------------------------------------------
void* dgr_hand_barrett3(int budget, std::uint64_t seed) {
  try { return new HandModel(make_three_finger_hand(budget, seed)); } catch (const std::exception& e) { fail(e); return nullptr; }
}
void* dgr_hand_pincher2(int budget, std::uint64_t seed) {
  try { return new HandModel(make_two_finger_hand(budget, seed)); } catch (const std::exception& e) { fail(e); return nullptr; }
}
void* dgr_hand_load_xml(const char* path, int budget, std::uint64_t seed) {
  try { return new HandModel(HandModel::load_xml(path, budget, seed)); } catch (const std::exception& e) { fail(e); return nullptr; }
}
void dgr_hand_free(void* h) { delete static_cast<HandModel*>(h); }

void dgr_hand_dims(void* hp, int* out) {
  auto* h = static_cast<HandModel*>(hp);
  out[0] = h->num_links();
  out[1] = h->num_joints();
  out[2] = h->total_samples();
}

// Descriptor in forward() order (hand.hpp:143-151): link-index major.
void dgr_hand_export(void* hp, int* topo, int* link_parent_joint, int* joint_parent, int* joint_child,
                     double* axis, double* origin_R, double* origin_t, double* lower, double* upper,
                     double* samples, int* sample_link) {
  auto* h = static_cast<HandModel*>(hp);
  std::vector<int> order = topo_order(*h);
  for (int i = 0; i < h->num_links(); ++i) {
    topo[i] = order[i];
    link_parent_joint[i] = h->links()[i].parent_joint;
  }
  for (int j = 0; j < h->num_joints(); ++j) {
    const HandJoint& jt = h->joints()[j];
    joint_parent[j] = jt.parent_link;
    joint_child[j] = jt.child_link;
    axis[3 * j] = jt.axis.x; axis[3 * j + 1] = jt.axis.y; axis[3 * j + 2] = jt.axis.z;
    for (int k = 0; k < 9; ++k) origin_R[9 * j + k] = jt.origin_R.m[k];
    origin_t[3 * j] = jt.origin_t.x; origin_t[3 * j + 1] = jt.origin_t.y; origin_t[3 * j + 2] = jt.origin_t.z;
    lower[j] = jt.lower;
    upper[j] = jt.upper;
  }
  int n = 0;
  for (int li = 0; li < h->num_links(); ++li)
    for (const Vec3& s : h->links()[li].samples) {
      samples[3 * n] = s.x; samples[3 * n + 1] = s.y; samples[3 * n + 2] = s.z;
      sample_link[n] = li;
      ++n;
    }
}

// per-sample surface area (HandModel::sample_areas, hand.hpp:77; link area /
// link sample count, hand.cpp:199-207), forward() order
void dgr_hand_sample_areas(void* hp, double* out) {
  const auto& a = static_cast<HandModel*>(hp)->sample_areas();
  for (std::size_t i = 0; i < a.size(); ++i) out[i] = a[i];
}

int dgr_hand_forward(void* hp, const double* q, double* out) {
  try {
    auto* h = static_cast<HandModel*>(hp);
    std::vector<Vec3> p = h->forward(unpack_q(*h, q));
    for (std::size_t i = 0; i < p.size(); ++i) { out[3 * i] = p[i].x; out[3 * i + 1] = p[i].y; out[3 * i + 2] = p[i].z; }
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// ---- objects --------------------------------------------------------------
void* dgr_object_mesh(const double* V, int nv, const int* F, int nf, double density, double alpha) {
  try {
    TriMesh m;
    for (int i = 0; i < nv; ++i) m.vertices.push_back({V[3 * i], V[3 * i + 1], V[3 * i + 2]});
    for (int f = 0; f < nf; ++f) m.faces.push_back({F[3 * f], F[3 * f + 1], F[3 * f + 2]});
    m.finalize();
    return new GraspObject(std::move(m), density, alpha);
  } catch (const std::exception& e) { fail(e); return nullptr; }
}
void* dgr_object_icosphere(double radius, int subdiv, double density, double alpha) {
  try { return new GraspObject(make_icosphere(radius, subdiv), density, alpha); } catch (const std::exception& e) { fail(e); return nullptr; }
}
void* dgr_object_box_mesh(double sx, double sy, double sz, double density, double alpha) {
  try { return new GraspObject(make_box(sx, sy, sz), density, alpha); } catch (const std::exception& e) { fail(e); return nullptr; }
}
void* dgr_object_cylinder_mesh(double radius, double height, int segments, double density, double alpha) {
  try { return new GraspObject(make_cylinder(radius, height, segments), density, alpha); } catch (const std::exception& e) { fail(e); return nullptr; }
}
void* dgr_object_blob_mesh(double radius, int subdiv, double amplitude, std::uint64_t seed, double density, double alpha) {
  try { return new GraspObject(make_blob(radius, subdiv, amplitude, seed), density, alpha); } catch (const std::exception& e) { fail(e); return nullptr; }
}
void dgr_object_free(void* o) { delete static_cast<GraspObject*>(o); }

// the object's TriMesh (vertices, faces, vertex normals) and alpha_phong
void dgr_object_mesh_dims(void* o, int* out) {
  const TriMesh& m = static_cast<GraspObject*>(o)->sdf.mesh();
  out[0] = static_cast<int>(m.num_vertices());
  out[1] = static_cast<int>(m.num_faces());
}
void dgr_object_mesh_export(void* o, double* V, int* F, double* VN) {
  const TriMesh& m = static_cast<GraspObject*>(o)->sdf.mesh();
  for (std::size_t i = 0; i < m.num_vertices(); ++i) {
    V[3 * i] = m.vertices[i].x; V[3 * i + 1] = m.vertices[i].y; V[3 * i + 2] = m.vertices[i].z;
    VN[3 * i] = m.vertex_normals[i].x; VN[3 * i + 1] = m.vertex_normals[i].y; VN[3 * i + 2] = m.vertex_normals[i].z;
  }
  for (std::size_t f = 0; f < m.num_faces(); ++f)
    for (int k = 0; k < 3; ++k) F[3 * f + k] = m.faces[f][k];
}

// the reference Bvh (bvh.hpp:27-33, 55-56): node boxes [n,6], (left, right,
// first, count) [n,4], face_order [F]; returns the node count
int dgr_object_bvh(void* o, double* boxes, int* links, int* face_order, int cap) {
  const MeshSdf& sdf = *static_cast<GraspObject*>(o)->sdf.mesh_sdf();
  const auto& nodes = sdf.bvh().nodes();
  const int n = static_cast<int>(nodes.size());
  for (int i = 0; i < n && i < cap; ++i) {
    const auto& nd = nodes[i];
    boxes[6 * i] = nd.box.lo.x; boxes[6 * i + 1] = nd.box.lo.y; boxes[6 * i + 2] = nd.box.lo.z;
    boxes[6 * i + 3] = nd.box.hi.x; boxes[6 * i + 4] = nd.box.hi.y; boxes[6 * i + 5] = nd.box.hi.z;
    links[4 * i] = nd.left; links[4 * i + 1] = nd.right; links[4 * i + 2] = nd.first; links[4 * i + 3] = nd.count;
  }
  const auto& fo = sdf.bvh().face_order();
  for (std::size_t i = 0; i < fo.size(); ++i) face_order[i] = fo[i];
  return n;
}

void dgr_object_use_sphere(void* o, double cx, double cy, double cz, double r) {
  static_cast<GraspObject*>(o)->sdf.use_sphere(dgx::SphereSdf{{cx, cy, cz}, r});
}
void dgr_object_use_box(void* o, const double* c, const double* h) {
  static_cast<GraspObject*>(o)->sdf.use_box(dgx::BoxSdf{{c[0], c[1], c[2]}, {h[0], h[1], h[2]}});
}
void dgr_object_use_grid(void* o, const int* dims, const double* origin, double h, double inv_h, const float* vals) {
  dgx::GridSdf g{dims[0], dims[1], dims[2], {origin[0], origin[1], origin[2]}, h, inv_h, nullptr, nullptr, 0,
                 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
  std::vector<float> v(vals, vals + static_cast<std::size_t>(dims[0]) * dims[1] * dims[2]);
  static_cast<GraspObject*>(o)->sdf.use_grid(g, std::move(v));
}

void dgr_object_set_inertial(void* o, double mass, const double* com, const double* I, const double* Iinv) {
  InertialData& in = static_cast<GraspObject*>(o)->inertial;
  in.mass = mass;
  in.com = {com[0], com[1], com[2]};
  for (int k = 0; k < 9; ++k) { in.inertia_body.m[k] = I[k]; in.inertia_body_inv.m[k] = Iinv[k]; }
}
void dgr_object_get_inertial(void* o, double* mass, double* com, double* I, double* Iinv) {
  const InertialData& in = static_cast<GraspObject*>(o)->inertial;
  *mass = in.mass;
  com[0] = in.com.x; com[1] = in.com.y; com[2] = in.com.z;
  for (int k = 0; k < 9; ++k) { I[k] = in.inertia_body.m[k]; Iinv[k] = in.inertia_body_inv.m[k]; }
}

// dilated query: out = rho, grad(3), proxy(3), sign
int dgr_object_query(void* o, const double* r, double radius, double* out) {
  try {
    PhongQuery q = static_cast<GraspObject*>(o)->sdf.dilated({r[0], r[1], r[2]}, radius);
    out[0] = q.rho;
    out[1] = q.grad.x; out[2] = q.grad.y; out[3] = q.grad.z;
    out[4] = q.smoothed_point.x; out[5] = q.smoothed_point.y; out[6] = q.smoothed_point.z;
    out[7] = q.sign;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// forward-only query MeshSdf::dilated_within (sdf.cpp:69-81) with the
// solver's cull margin (sim.hpp:213); nullopt -> out[0] = +inf, rest 0
int dgr_object_query_within(void* o, const double* r, double radius, double* out) {
  try {
    auto q = static_cast<GraspObject*>(o)->sdf.dilated_within({r[0], r[1], r[2]}, radius, 0.005);
    if (!q) {
      out[0] = std::numeric_limits<double>::infinity();
      for (int k = 1; k < 8; ++k) out[k] = 0.0;
      return 0;
    }
    out[0] = q->rho;
    out[1] = q->grad.x; out[2] = q->grad.y; out[3] = q->grad.z;
    out[4] = q->smoothed_point.x; out[5] = q->smoothed_point.y; out[6] = q->smoothed_point.z;
    out[7] = q->sign;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// ---- scene drop -------------------------------------------
// The reference's step_on_table (sim.cpp:14-94) iterated on one RigidState
// with the driver rule of dgx_drop_batch: stop once settle consecutive steps
// made contact (any correction) and left kinetic_energy (sim.cpp:8-12) <
// ke_tol, never before min_steps, at most max_steps. One SolveStats shared by
// all steps.
int dgr_drop(void* o, const double* in, double dt, double mu, int gs, const double* gravity, int max_steps,
             int min_steps, double ke_tol, int measure, double* out, int* steps, double* ke, double* stats,
             double* traj, int record_every, int settle) {
  try {
    const auto& obj = *static_cast<GraspObject*>(o);
    SimParams p;
    p.dt = dt;
    p.mu = mu;
    p.gs_iters = gs;
    p.gravity = Vec3{gravity[0], gravity[1], gravity[2]};
    RigidState s;
    s.x = {in[0], in[1], in[2]};
    s.theta = {in[3], in[4], in[5], in[6]};
    s.xdot = {in[7], in[8], in[9]};
    s.thetadot = {in[10], in[11], in[12]};
    SolveStats st;
    st.measure_residual = measure != 0;
    int k = 0, calm = 0;
    double e = kinetic_energy(s, obj.inertial);
    for (; k < max_steps;) {
      const int corr_before = st.corrections;
      s = step_on_table(s, obj.sdf.mesh(), obj.inertial, p, &st);
      ++k;
      if (traj && record_every > 0 && k % record_every == 0) {
        double* t = traj + static_cast<std::size_t>(k / record_every - 1) * 13;
        t[0] = s.x.x; t[1] = s.x.y; t[2] = s.x.z;
        t[3] = s.theta.w; t[4] = s.theta.x; t[5] = s.theta.y; t[6] = s.theta.z;
        t[7] = s.xdot.x; t[8] = s.xdot.y; t[9] = s.xdot.z;
        t[10] = s.thetadot.x; t[11] = s.thetadot.y; t[12] = s.thetadot.z;
      }
      e = kinetic_energy(s, obj.inertial);
      calm = (st.corrections > corr_before && e < ke_tol) ? calm + 1 : 0;
      if (calm >= settle && k >= min_steps) break;
    }
    out[0] = s.x.x; out[1] = s.x.y; out[2] = s.x.z;
    out[3] = s.theta.w; out[4] = s.theta.x; out[5] = s.theta.y; out[6] = s.theta.z;
    out[7] = s.xdot.x; out[8] = s.xdot.y; out[9] = s.xdot.z;
    out[10] = s.thetadot.x; out[11] = s.thetadot.y; out[12] = s.thetadot.z;
    *steps = k;
    *ke = e;
    stats[0] = st.active_contacts; stats[1] = st.corrections; stats[2] = st.singular_skipped;
    stats[3] = st.max_penetration;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// ---- objective ------------------------------------------------------------
int dgr_loss_gradient(void* o, void* hp, const double* q, const Params* p, double* losses,
                      double* d_stable, double* d_qrange, double* d_qlimit) {
  try {
    auto* h = static_cast<HandModel*>(hp);
    LossGradient g = loss_gradient(*static_cast<GraspObject*>(o), *h, unpack_q(*h, q), protocol(*p), sim_params(*p));
    losses[0] = g.losses.stable; losses[1] = g.losses.qrange; losses[2] = g.losses.qlimit;
    std::copy(g.d_stable.begin(), g.d_stable.end(), d_stable);
    std::copy(g.d_qrange.begin(), g.d_qrange.end(), d_qrange);
    std::copy(g.d_qlimit.begin(), g.d_qlimit.end(), d_qlimit);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int dgr_evaluate_losses(void* o, void* hp, const double* q, const Params* p, double* losses) {
  try {
    auto* h = static_cast<HandModel*>(hp);
    LossBreakdown b = evaluate_losses(*static_cast<GraspObject*>(o), *h, unpack_q(*h, q), protocol(*p), sim_params(*p));
    losses[0] = b.stable; losses[1] = b.qrange; losses[2] = b.qlimit;
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

int dgr_apply_gradient_step(void* hp, const double* q, const double* g, double lr, double* q_out) {
  try {
    auto* h = static_cast<HandModel*>(hp);
    std::vector<double> gv(g, g + 6 + h->num_joints());
    pack_q(apply_gradient_step(unpack_q(*h, q), gv, lr), q_out);
    return 0;
  } catch (const std::exception& e) { return fail(e); }
}

// One recorded perturbation sim (losses.cpp:32-42): residual, its tape
// gradient (6+J), optional d residual / d p_i (points as tape inputs, N*3),
// and the rho_d of every SDF call in call order (sweep-major, point-minor).
// debug (multi-step protocols): d residual / d (state after step 1) of a
// two-step perturbation sim, the reference tape with the step-1 state
// re-registered as 13 inputs (x 3, theta w,x,y,z 4, xdot 3, thetadot 3)
int dgr_debug_step_adjoint(void* o, void* hp, const double* q, int m, const Params* p, double* out) {
  try {
    auto* h = static_cast<HandModel*>(hp);
    const auto& obj = *static_cast<GraspObject*>(o);
    StabilityProtocol proto = protocol(*p);
    SimParams sim = sim_params(*p);
    sim.gravity = Vec3{};
    HandConfig cfg = unpack_q(*h, q);
    std::vector<Vec3> pts = h->forward(cfg);
    // step 1 on values
    BodyStateT<double> s0 = to_body_state<double>(canonical_state(obj.inertial));
    s0.xdot = proto.velocities[m];
    BodyStateT<double> s1 = step(s0, pts, obj.sdf, obj.inertial, sim);
    Tape tape;
    Tape::Scope scope(tape);
    std::vector<Vec3T<Rec>> rp;
    for (const Vec3& v : pts) rp.push_back({Rec(v.x), Rec(v.y), Rec(v.z)});
    BodyStateT<Rec> r1;
    r1.x = {tape.input(s1.x.x), tape.input(s1.x.y), tape.input(s1.x.z)};
    r1.theta = {tape.input(s1.theta.w), tape.input(s1.theta.x), tape.input(s1.theta.y), tape.input(s1.theta.z)};
    r1.xdot = {tape.input(s1.xdot.x), tape.input(s1.xdot.y), tape.input(s1.xdot.z)};
    r1.thetadot = {tape.input(s1.thetadot.x), tape.input(s1.thetadot.y), tape.input(s1.thetadot.z)};
    BodyStateT<double> pd = predict(s1, sim);
    BodyStateT<Rec> rpd;  // the predicted state as separate inputs (13 more)
    rpd.x = {tape.input(pd.x.x), tape.input(pd.x.y), tape.input(pd.x.z)};
    rpd.theta = {tape.input(pd.theta.w), tape.input(pd.theta.x), tape.input(pd.theta.y), tape.input(pd.theta.z)};
    rpd.xdot = {tape.input(pd.xdot.x), tape.input(pd.xdot.y), tape.input(pd.xdot.z)};
    rpd.thetadot = {tape.input(pd.thetadot.x), tape.input(pd.thetadot.y), tape.input(pd.thetadot.z)};
    BodyStateT<Rec> r2 = solve_contacts(r1, rpd, rp, obj.sdf, obj.inertial, sim);
    Rec res = norm(r2.xdot) + norm(r2.thetadot);
    tape.set_output(res);
    std::vector<double> g = tape.gradient();
    std::copy(g.begin(), g.begin() + 26, out);  // d/d prev (13), d/d pred (13)
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int dgr_sim_record(void* o, void* hp, const double* q, int m, const Params* p, double* residual,
                   double* grad, double* grad_points, double* rho_log, int rho_cap, int* n_calls) {
  try {
    auto* h = static_cast<HandModel*>(hp);
    const auto& obj = *static_cast<GraspObject*>(o);
    StabilityProtocol proto = protocol(*p);
    SimParams sim = sim_params(*p);
    sim.gravity = Vec3{};
    HandConfig cfg = unpack_q(*h, q);
    std::vector<double> log;
    g_trace.rho = &log;
    {
      Tape tape;
      Tape::Scope scope(tape);
      Rec r = recorded_residual(obj, *h, cfg, proto, sim, m, tape, nullptr);
      tape.set_output(r);
      *residual = r.v;
      if (grad) {
        std::vector<double> g = tape.gradient();
        std::copy(g.begin(), g.end(), grad);
      }
    }
    g_trace.rho = nullptr;
    if (grad_points) {
      // same sim with the world points themselves registered as inputs
      std::vector<Vec3> pts = h->forward(cfg);
      Tape tape;
      Tape::Scope scope(tape);
      std::vector<Vec3T<Rec>> rp;
      rp.reserve(pts.size());
      for (const Vec3& v : pts) rp.push_back({tape.input(v.x), tape.input(v.y), tape.input(v.z)});
      Rec r = perturbation_residual(obj, rp, proto.velocities[m], proto, sim);
      tape.set_output(r);
      std::vector<double> g = tape.gradient();
      std::copy(g.begin(), g.end(), grad_points);
    }
    if (n_calls) *n_calls = static_cast<int>(log.size());
    if (rho_log) std::copy(log.begin(), log.begin() + std::min<std::size_t>(log.size(), rho_cap), rho_log);
    return 0;
  } catch (const std::exception& e) {
    g_trace.rho = nullptr;
    return fail(e);
  }
}

// Forward-only (double) perturbation sim with SolveStats (sim.hpp:42-49), as
// perturbation_residual<double> (losses.hpp:47-57) with the stats plumbed
// through; stats = active_contacts, corrections, singular_skipped,
// max_penetration, max_friction_ratio. Also logs every SDF query.
int dgr_sim_forward(void* o, void* hp, const double* q, int m, const Params* p, int measure_residual,
                    double* residual, double* stats, double* rho_log, int rho_cap, int* n_calls) {
  try {
    auto* h = static_cast<HandModel*>(hp);
    const auto& obj = *static_cast<GraspObject*>(o);
    StabilityProtocol proto = protocol(*p);
    SimParams sim = sim_params(*p);
    sim.gravity = Vec3{};
    std::vector<Vec3> pts = h->forward(unpack_q(*h, q));
    std::vector<double> log;
    g_trace.rho = &log;
    SolveStats st;
    st.measure_residual = measure_residual != 0;
    BodyStateT<double> s = to_body_state<double>(canonical_state(obj.inertial));
    const Vec3& v = proto.velocities[m];
    s.xdot = {v.x, v.y, v.z};
    for (int t = 0; t < proto.steps; ++t) s = step(s, pts, obj.sdf, obj.inertial, sim, &st);
    g_trace.rho = nullptr;
    *residual = norm(s.xdot) + norm(s.thetadot);
    stats[0] = st.active_contacts; stats[1] = st.corrections; stats[2] = st.singular_skipped;
    stats[3] = st.max_penetration; stats[4] = st.max_friction_ratio;
    if (n_calls) *n_calls = static_cast<int>(log.size());
    if (rho_log) std::copy(log.begin(), log.begin() + std::min<std::size_t>(log.size(), rho_cap), rho_log);
    return 0;
  } catch (const std::exception& e) {
    g_trace.rho = nullptr;
    return fail(e);
  }
}

// Shared synthesis driver, candidates split over `threads`
// std::threads. For k in [k_begin, k_end): r_k = r0*(1 - k/(K-1)) (0 when
// K == 1); loss_gradient at r_k; g = weighted(w) (losses.hpp:110-115); Adam
// (t = k+1, bias corrections from running products of beta); q <-
// apply_gradient_step(q, adam_dir, lr) (losses.cpp:92-102). q, adam_m, adam_v
// are updated in place. Optional per-iteration records (k_end-k_begin rows per
// candidate): losses (3) and the weighted gradient (6+J) at the iterate.
int dgr_optimize(void* o, void* hp, int B, double* q, double* adam_m, double* adam_v, const Params* p,
                 const OptCfg* cfg, int threads, double* traj_losses, double* traj_grads, int* status) {
  auto* h = static_cast<HandModel*>(hp);
  const auto& obj = *static_cast<GraspObject*>(o);
  const int J = h->num_joints(), D = 6 + J, Q = 7 + J;
  const int steps = cfg->k_end - cfg->k_begin;
  StabilityProtocol proto = protocol(*p);
  LossWeights w{p->w_stable, p->w_qrange, p->w_qlimit};
  std::atomic<int> next{0};
  auto worker = [&]() {
    for (;;) {
      int b = next.fetch_add(1);
      if (b >= B) return;
      try {
        HandConfig c = unpack_q(*h, q + static_cast<std::size_t>(b) * Q);
        double* mm = adam_m + static_cast<std::size_t>(b) * D;
        double* vv = adam_v + static_cast<std::size_t>(b) * D;
        double b1t = 1.0, b2t = 1.0;
        for (int k = 0; k < cfg->k_begin; ++k) { b1t *= cfg->beta1; b2t *= cfg->beta2; }
        for (int k = cfg->k_begin; k < cfg->k_end; ++k) {
          SimParams sim = sim_params(*p);
          sim.dilation_radius =
              cfg->iters > 1 ? cfg->r0 * (1.0 - static_cast<double>(k) / static_cast<double>(cfg->iters - 1)) : 0.0;
          LossGradient lg = loss_gradient(obj, *h, c, proto, sim);
          std::vector<double> g = lg.weighted(w);
          for (double gi : g)
            if (!std::isfinite(gi)) throw std::runtime_error("non-finite gradient");
          if (traj_losses) {
            double* tl = traj_losses + (static_cast<std::size_t>(b) * steps + (k - cfg->k_begin)) * 3;
            tl[0] = lg.losses.stable; tl[1] = lg.losses.qrange; tl[2] = lg.losses.qlimit;
          }
          if (traj_grads)
            std::copy(g.begin(), g.end(), traj_grads + (static_cast<std::size_t>(b) * steps + (k - cfg->k_begin)) * D);
          b1t *= cfg->beta1;
          b2t *= cfg->beta2;
          const double c1 = 1.0 - cfg->beta1, c2 = 1.0 - cfg->beta2;
          std::vector<double> dir(D);
          for (int i = 0; i < D; ++i) {
            mm[i] = cfg->beta1 * mm[i] + c1 * g[i];
            vv[i] = cfg->beta2 * vv[i] + c2 * (g[i] * g[i]);
            double mhat = mm[i] / (1.0 - b1t);
            double vhat = vv[i] / (1.0 - b2t);
            dir[i] = mhat / (std::sqrt(vhat) + cfg->eps);
          }
          c = apply_gradient_step(c, dir, cfg->lr);
        }
        pack_q(c, q + static_cast<std::size_t>(b) * Q);
        status[b] = 0;
      } catch (const std::exception&) {
        status[b] = 1;
      }
    }
  };
  int nt = std::max(1, threads);
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  return 0;
}

}  // extern "C"
