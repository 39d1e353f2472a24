// include/dgx/diffgrasp.hpp — drop-in C++ API over libdgx_cuda.so for code
// written against the reference library (/root/reference/proj/include/
// diffgrasp). Header-only; needs the reference headers on the include path
// (it consumes dg:: types) and links -ldgx_cuda.
//
// Mapping (reference -> here), same argument meaning, same exception types
// and messages:
//   dg::HandModel::forward(const HandConfig&)      hand.hpp:86      -> dgx::forward
//   dg::loss_gradient(obj, hand, q, proto, params) losses.hpp:126   -> dgx::loss_gradient
//   dg::evaluate_losses(obj, hand, q, proto, params) losses.hpp:119 -> dgx::evaluate_losses
//   dg::apply_gradient_step(q, grad, lr)           losses.hpp:136   -> dgx::apply_gradient_step
// plus batched overloads over std::span<const dg::HandConfig> and the fused
// synthesis loop dgx::optimize (the reference has none).
// The reference's exact signatures (no Runtime / handles: a per-thread
// runtime and upload cache) are at the end of this header:
//   dgx::loss_gradient(obj, hand, q, proto, params)   == dg::loss_gradient
//   dgx::evaluate_losses(obj, hand, q, proto, params) == dg::evaluate_losses
//   dgx::apply_gradient_step(q, grad, lr)             == dg::apply_gradient_step
//   dgx::forward(hand, q)                             == hand.forward(q)
//
// The object: dgx::Object(rt, const dg::GraspObject&) takes the reference's
// own object (losses.hpp:38-44) unchanged: its TriMesh (vertices, faces,
// vertex normals), MeshSdf alpha_phong and InertialData; queries are the
// reference's MeshSdf ones (csrc/dgx_mesh.h). dgx::Object(rt, SdfSpec,
// InertialData) adds the analytic / grid backends the reference lacks.
//   dg::MeshSdf::dilated / dilated_within        sdf.hpp:41-45   -> dgx::dilated / dilated_within
#pragma once

#include <cstdint>
#include <cstdlib>
#include <limits>
#include <memory>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "diffgrasp/hand.hpp"
#include "diffgrasp/losses.hpp"
#include "diffgrasp/rigid.hpp"
#include "diffgrasp/sim.hpp"
#include "dgx.h"

namespace dgx {

namespace detail {
inline void check(int rc) {
  if (rc == DGX_OK) return;
  const std::string msg = dgx_last_error();
  if (rc == DGX_E_INVALID && msg.find("dilation radius") != std::string::npos) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
// per-candidate status -> the reference's exception (losses.cpp:15-16, tape.cpp:35-38)
inline void check_candidate(int32_t st) {
  switch (st) {
    case DGX_OK: return;
    case DGX_E_NONFINITE_LOSS: throw std::runtime_error("loss evaluation produced a non-finite value");
    case DGX_E_NONFINITE_GRAD: throw std::runtime_error("tape: non-finite adjoint");
    default: throw std::runtime_error("dgx: candidate failed with status " + std::to_string(st));
  }
}
inline std::vector<double> pack(const dg::HandConfig& q) {
  std::vector<double> v{q.base_position.x, q.base_position.y, q.base_position.z, q.base_orientation.w,
                        q.base_orientation.x, q.base_orientation.y, q.base_orientation.z};
  v.insert(v.end(), q.joint_angles.begin(), q.joint_angles.end());
  return v;
}
inline dg::HandConfig unpack(const double* v, int J) {
  dg::HandConfig q;
  q.base_position = {v[0], v[1], v[2]};
  q.base_orientation = {v[3], v[4], v[5], v[6]};
  q.joint_angles.assign(v + 7, v + 7 + J);
  return q;
}
inline dgx_params params_of(const dg::StabilityProtocol& proto, const dg::SimParams& p,
                            const dg::LossWeights& w = {}) {
  static_assert(sizeof(dg::Vec3) == 3 * sizeof(double), "dg::Vec3 must be three packed doubles");
  dgx_params c{};
  c.dt = p.dt;
  c.mu = p.mu;
  c.gs_iters = p.gs_iters;
  c.steps = proto.steps;
  c.dilation_radius = p.dilation_radius;
  c.alpha_leak = p.leak.alpha_leak;
  c.num_velocities = proto.m();
  for (int m = 0; m < proto.m() && m < 8; ++m) {
    c.velocities[m][0] = proto.velocities[m].x;
    c.velocities[m][1] = proto.velocities[m].y;
    c.velocities[m][2] = proto.velocities[m].z;
  }
  // any M (losses.hpp:17): the protocol's own vector, alive for the call
  if (proto.m() > 8) c.velocity_list = reinterpret_cast<const double*>(proto.velocities.data());
  c.w_stable = w.stable;
  c.w_qrange = w.qrange;
  c.w_qlimit = w.qlimit;
  return c;
}
}  // namespace detail

// One device + stream.
class Runtime {
 public:
  explicit Runtime(int device = 0) { detail::check(dgx_ctx_create(device, &ctx_)); }
  ~Runtime() { dgx_ctx_destroy(ctx_); }
  Runtime(const Runtime&) = delete;
  Runtime& operator=(const Runtime&) = delete;
  dgx_ctx* get() const { return ctx_; }

 private:
  dgx_ctx* ctx_ = nullptr;
};

// A dg::HandModel resident on the device (samples in forward() order).
class Hand {
 public:
  Hand(Runtime& rt, const dg::HandModel& h) : J_(h.num_joints()), N_(h.total_samples()) {
    const int L = h.num_links();
    std::vector<int32_t> topo{h.base_link()}, lpj(L), jp(J_), jc(J_), sl;
    for (std::size_t head = 0; head < topo.size(); ++head)  // BFS of hand.cpp:177-194
      for (int j = 0; j < J_; ++j)
        if (h.joints()[j].parent_link == topo[head]) topo.push_back(h.joints()[j].child_link);
    std::vector<double> axis, oR, ot, lo, up, smp;
    for (int l = 0; l < L; ++l) lpj[l] = h.links()[l].parent_joint;
    for (int j = 0; j < J_; ++j) {
      const auto& jt = h.joints()[j];
      jp[j] = jt.parent_link;
      jc[j] = jt.child_link;
      axis.insert(axis.end(), {jt.axis.x, jt.axis.y, jt.axis.z});
      oR.insert(oR.end(), jt.origin_R.m.begin(), jt.origin_R.m.end());
      ot.insert(ot.end(), {jt.origin_t.x, jt.origin_t.y, jt.origin_t.z});
      lo.push_back(jt.lower);
      up.push_back(jt.upper);
    }
    for (int l = 0; l < L; ++l)
      for (const auto& s : h.links()[l].samples) {
        smp.insert(smp.end(), {s.x, s.y, s.z});
        sl.push_back(l);
      }
    dgx_hand_desc d{L, J_, N_, topo.data(), lpj.data(), jp.data(), jc.data(), axis.data(), oR.data(), ot.data(),
                    lo.data(), up.data(), smp.data(), sl.data()};
    detail::check(dgx_hand_upload(rt.get(), &d, &h_));
  }
  ~Hand() { dgx_hand_free(h_); }
  Hand(const Hand&) = delete;
  Hand& operator=(const Hand&) = delete;
  const dgx_hand* get() const { return h_; }
  int num_joints() const { return J_; }
  int num_samples() const { return N_; }

 private:
  dgx_hand* h_ = nullptr;
  int J_, N_;
};

// SDF backend description (csrc/dgx_geom.h): sphere, box, or FP32 grid.
struct SdfSpec {
  int kind = DGX_SDF_SPHERE;
  double center[3] = {0, 0, 0};
  double radius = 0.0;
  double half_extents[3] = {0, 0, 0};
  int dims[3] = {0, 0, 0};
  double origin[3] = {0, 0, 0};
  double spacing = 0.0, inv_spacing = 0.0;
  std::vector<float> values;
};

class Object {
 public:
  Object(Runtime& rt, const SdfSpec& s, const dg::InertialData& in) {
    dgx_object_desc d{};
    d.kind = s.kind;
    for (int k = 0; k < 3; ++k) {
      d.center[k] = s.center[k];
      d.half_extents[k] = s.half_extents[k];
      d.dims[k] = s.dims[k];
      d.origin[k] = s.origin[k];
    }
    d.radius = s.radius;
    d.spacing = s.spacing;
    d.inv_spacing = s.inv_spacing;
    d.values = s.values.empty() ? nullptr : s.values.data();
    d.mass = in.mass;
    d.com[0] = in.com.x; d.com[1] = in.com.y; d.com[2] = in.com.z;
    for (int k = 0; k < 9; ++k) d.inertia_body_inv[k] = in.inertia_body_inv.m[k];
    detail::check(dgx_object_upload(rt.get(), &d, &o_));
  }
  // dg::GraspObject (mesh SDF + InertialData) as the reference builds it
  Object(Runtime& rt, const dg::GraspObject& go) {
    const dg::TriMesh& m = go.sdf.mesh();
    std::vector<double> V(3 * m.num_vertices()), VN(3 * m.num_vertices());
    std::vector<int32_t> F(3 * m.num_faces());
    for (std::size_t i = 0; i < m.num_vertices(); ++i) {
      V[3 * i] = m.vertices[i].x; V[3 * i + 1] = m.vertices[i].y; V[3 * i + 2] = m.vertices[i].z;
      VN[3 * i] = m.vertex_normals[i].x; VN[3 * i + 1] = m.vertex_normals[i].y; VN[3 * i + 2] = m.vertex_normals[i].z;
    }
    for (std::size_t f = 0; f < m.num_faces(); ++f)
      for (int k = 0; k < 3; ++k) F[3 * f + k] = m.faces[f][k];
    dgx_object_desc d{};
    d.kind = DGX_SDF_MESH;
    d.num_vertices = static_cast<int32_t>(m.num_vertices());
    d.num_faces = static_cast<int32_t>(m.num_faces());
    d.vertices = V.data();
    d.faces = F.data();
    d.vertex_normals = VN.data();
    d.alpha_phong = go.sdf.alpha_phong();
    const dg::InertialData& in = go.inertial;
    d.mass = in.mass;
    d.com[0] = in.com.x; d.com[1] = in.com.y; d.com[2] = in.com.z;
    for (int k = 0; k < 9; ++k) d.inertia_body_inv[k] = in.inertia_body_inv.m[k];
    detail::check(dgx_object_upload(rt.get(), &d, &o_));
  }
  ~Object() { dgx_object_free(o_); }
  Object(const Object&) = delete;
  Object& operator=(const Object&) = delete;
  const dgx_object* get() const { return o_; }

 private:
  dgx_object* o_ = nullptr;
};

// ---- SDF queries (MeshSdf::dilated / dilated_within, sdf.hpp:41-45) ----------
// Batched over object-frame points; PhongQuery::flat is not reported.
inline std::vector<std::optional<dg::PhongQuery>> sdf_queries(Runtime& rt, const Object& obj,
                                                              std::span<const dg::Vec3> r, double radius,
                                                              bool within) {
  std::vector<double> p(3 * r.size()), out(8 * r.size());
  for (std::size_t i = 0; i < r.size(); ++i) { p[3 * i] = r[i].x; p[3 * i + 1] = r[i].y; p[3 * i + 2] = r[i].z; }
  detail::check(dgx_sdf_query_batch(rt.get(), obj.get(), static_cast<int32_t>(r.size()), p.data(), radius,
                                    within ? 1 : 0, out.data(), 0));
  std::vector<std::optional<dg::PhongQuery>> res(r.size());
  for (std::size_t i = 0; i < r.size(); ++i) {
    const double* o = out.data() + 8 * i;
    if (o[7] == 0.0) continue;  // culled (nullopt)
    dg::PhongQuery q;
    q.rho = o[0];
    q.grad = {o[1], o[2], o[3]};
    q.smoothed_point = {o[4], o[5], o[6]};
    q.sign = static_cast<int>(o[7]);
    res[i] = q;
  }
  return res;
}
inline dg::PhongQuery dilated(Runtime& rt, const Object& obj, const dg::Vec3& r, double radius) {
  return *sdf_queries(rt, obj, std::span<const dg::Vec3>(&r, 1), radius, false)[0];
}
// with the solver's cull margin (sim.hpp:213)
inline std::optional<dg::PhongQuery> dilated_within(Runtime& rt, const Object& obj, const dg::Vec3& r, double radius) {
  return sdf_queries(rt, obj, std::span<const dg::Vec3>(&r, 1), radius, true)[0];
}

// ---- reference signatures (batch of one) ------------------------------------

inline std::vector<dg::Vec3> forward(Runtime& rt, const Hand& hand, const dg::HandConfig& q) {
  if (static_cast<int>(q.joint_angles.size()) != hand.num_joints())
    throw std::runtime_error("hand: expected " + std::to_string(hand.num_joints()) + " joint angles, got " +
                             std::to_string(q.joint_angles.size()));
  std::vector<double> qv = detail::pack(q), pts(3 * static_cast<std::size_t>(hand.num_samples()));
  detail::check(dgx_forward_batch(rt.get(), hand.get(), 1, qv.data(), pts.data(), 0));
  std::vector<dg::Vec3> out(hand.num_samples());
  for (int i = 0; i < hand.num_samples(); ++i) out[i] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
  return out;
}

inline std::vector<dg::LossGradient> loss_gradient(Runtime& rt, const Object& obj, const Hand& hand,
                                                   std::span<const dg::HandConfig> qs,
                                                   const dg::StabilityProtocol& proto, const dg::SimParams& params) {
  const int B = static_cast<int>(qs.size()), J = hand.num_joints(), D = 6 + J;
  std::vector<double> q;
  for (const auto& c : qs) {
    if (static_cast<int>(c.joint_angles.size()) != J) throw std::runtime_error("hand: joint angle count mismatch");
    auto v = detail::pack(c);
    q.insert(q.end(), v.begin(), v.end());
  }
  std::vector<double> losses(3 * static_cast<std::size_t>(B)), grads(3 * static_cast<std::size_t>(B) * D);
  std::vector<int32_t> status(B);
  const dgx_params p = detail::params_of(proto, params);
  detail::check(dgx_loss_gradient_batch(rt.get(), hand.get(), obj.get(), B, q.data(), &p, losses.data(),
                                        grads.data(), status.data(), 0));
  std::vector<dg::LossGradient> out(B);
  for (int b = 0; b < B; ++b) {
    detail::check_candidate(status[b]);
    out[b].losses = {losses[3 * b], losses[3 * b + 1], losses[3 * b + 2]};
    const double* g = grads.data() + static_cast<std::size_t>(b) * 3 * D;
    out[b].d_stable.assign(g, g + D);
    out[b].d_qrange.assign(g + D, g + 2 * D);
    out[b].d_qlimit.assign(g + 2 * D, g + 3 * D);
  }
  return out;
}

inline dg::LossGradient loss_gradient(Runtime& rt, const Object& obj, const Hand& hand, const dg::HandConfig& q,
                                      const dg::StabilityProtocol& proto, const dg::SimParams& params) {
  return loss_gradient(rt, obj, hand, std::span<const dg::HandConfig>(&q, 1), proto, params)[0];
}

inline dg::LossBreakdown evaluate_losses(Runtime& rt, const Object& obj, const Hand& hand, const dg::HandConfig& q,
                                         const dg::StabilityProtocol& proto, const dg::SimParams& params) {
  std::vector<double> qv = detail::pack(q), losses(3);
  int32_t status = 0;
  const dgx_params p = detail::params_of(proto, params);
  detail::check(dgx_evaluate_losses_batch(rt.get(), hand.get(), obj.get(), 1, qv.data(), &p, losses.data(),
                                          nullptr, &status, 0));
  detail::check_candidate(status);
  return {losses[0], losses[1], losses[2]};
}

inline dg::HandConfig apply_gradient_step(Runtime& rt, const Hand& hand, const dg::HandConfig& q,
                                          const std::vector<double>& grad, double lr) {
  std::vector<double> qv = detail::pack(q), out(qv.size());
  detail::check(dgx_apply_gradient_step_batch(rt.get(), hand.get(), 1, qv.data(), grad.data(), lr, out.data(), 0));
  return detail::unpack(out.data(), hand.num_joints());
}

// Fused synthesis loop over a batch: returns the final configs.
struct OptimizeConfig {
  int iterations = 200;
  double dilation_start_radius = 0.02, learning_rate = 1e-3, beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
};

inline std::vector<dg::HandConfig> optimize(Runtime& rt, const Object& obj, const Hand& hand,
                                            std::span<const dg::HandConfig> init, const dg::StabilityProtocol& proto,
                                            const dg::SimParams& params, const dg::LossWeights& w,
                                            const OptimizeConfig& cfg) {
  const int B = static_cast<int>(init.size()), J = hand.num_joints(), D = 6 + J;
  std::vector<double> q;
  for (const auto& c : init) {
    auto v = detail::pack(c);
    q.insert(q.end(), v.begin(), v.end());
  }
  std::vector<double> m(static_cast<std::size_t>(B) * D, 0.0), v(static_cast<std::size_t>(B) * D, 0.0);
  std::vector<int32_t> status(B);
  const dgx_params p = detail::params_of(proto, params, w);
  const dgx_opt o{cfg.iterations, 0, cfg.iterations, 0, cfg.dilation_start_radius, cfg.learning_rate, cfg.beta1,
                  cfg.beta2, cfg.eps};
  detail::check(dgx_optimize_batch(rt.get(), hand.get(), obj.get(), B, q.data(), m.data(), v.data(), &p, &o, nullptr,
                                   status.data(), 0));
  std::vector<dg::HandConfig> out;
  for (int b = 0; b < B; ++b) {
    detail::check_candidate(status[b]);
    out.push_back(detail::unpack(q.data() + static_cast<std::size_t>(b) * (7 + J), J));
  }
  return out;
}

// ---- true drop-in: the reference's own signatures ---------------------------
// Same argument lists as dg::loss_gradient / dg::evaluate_losses
// (losses.hpp:119-127), dg::apply_gradient_step (losses.hpp:136) and
// HandModel::forward (hand.hpp:86): a call site switches namespace
// (dg:: -> dgx::) and nothing else. The device runtime is per host thread
// (device DGX_DEVICE, default 0; the reference's tape is per thread too,
// tape.hpp:124), and uploads are cached per thread keyed on the object's /
// hand's address plus a content fingerprint, so a destroyed-and-rebuilt
// object at the same address is uploaded again.
namespace detail {
inline Runtime& thread_runtime() {
  thread_local Runtime rt([] {
    const char* ev = std::getenv("DGX_DEVICE");
    return ev ? std::atoi(ev) : 0;
  }());
  return rt;
}
inline uint64_t fnv(uint64_t h, const void* p, std::size_t n) {
  const unsigned char* c = static_cast<const unsigned char*>(p);
  for (std::size_t i = 0; i < n; ++i) h = (h ^ c[i]) * 1099511628211ull;
  return h;
}
inline uint64_t fingerprint(const dg::HandModel& h) {
  uint64_t f = 1469598103934665603ull;
  const int ints[3] = {h.num_links(), h.num_joints(), h.total_samples()};
  f = fnv(f, ints, sizeof ints);
  for (const auto& l : h.links())
    if (!l.samples.empty()) f = fnv(f, l.samples.data(), l.samples.size() * sizeof(dg::Vec3));
  for (const auto& j : h.joints()) {
    f = fnv(f, &j.axis, sizeof j.axis);
    f = fnv(f, &j.origin_t, sizeof j.origin_t);
    f = fnv(f, j.origin_R.m.data(), sizeof(double) * 9);
    f = fnv(f, &j.lower, sizeof j.lower);
    f = fnv(f, &j.upper, sizeof j.upper);
  }
  return f;
}
inline uint64_t fingerprint(const dg::GraspObject& o) {
  uint64_t f = 1469598103934665603ull;
  const dg::TriMesh& m = o.sdf.mesh();
  f = fnv(f, m.vertices.data(), m.vertices.size() * sizeof(dg::Vec3));
  f = fnv(f, m.faces.data(), m.faces.size() * sizeof(m.faces[0]));
  const double a = o.sdf.alpha_phong();
  f = fnv(f, &a, sizeof a);
  f = fnv(f, &o.inertial.mass, sizeof o.inertial.mass);
  f = fnv(f, &o.inertial.com, sizeof o.inertial.com);
  f = fnv(f, o.inertial.inertia_body_inv.m.data(), sizeof(double) * 9);
  return f;
}
template <class Dev, class Src>
struct UploadCache {
  struct Entry {
    const Src* key;
    uint64_t fp;
    std::unique_ptr<Dev> dev;
  };
  std::vector<Entry> entries;
  const Dev& get(const Src& s) {
    const uint64_t fp = fingerprint(s);
    for (auto& e : entries)
      if (e.key == &s) {
        if (e.fp != fp) {
          e.dev = std::make_unique<Dev>(thread_runtime(), s);
          e.fp = fp;
        }
        return *e.dev;
      }
    if (entries.size() >= 64) entries.erase(entries.begin());
    entries.push_back({&s, fp, std::make_unique<Dev>(thread_runtime(), s)});
    return *entries.back().dev;
  }
};
inline const Hand& cached(const dg::HandModel& h) {
  thread_local UploadCache<Hand, dg::HandModel> c;
  return c.get(h);
}
inline const Object& cached(const dg::GraspObject& o) {
  thread_local UploadCache<Object, dg::GraspObject> c;
  return c.get(o);
}
}  // namespace detail

// dg::loss_gradient (losses.hpp:126-127)
inline dg::LossGradient loss_gradient(const dg::GraspObject& object, const dg::HandModel& hand,
                                      const dg::HandConfig& q, const dg::StabilityProtocol& protocol,
                                      const dg::SimParams& params) {
  if (static_cast<int>(q.joint_angles.size()) != hand.num_joints())
    throw std::runtime_error("hand: expected " + std::to_string(hand.num_joints()) + " joint angles, got " +
                             std::to_string(q.joint_angles.size()));
  return loss_gradient(detail::thread_runtime(), detail::cached(object), detail::cached(hand), q, protocol, params);
}

// dg::evaluate_losses (losses.hpp:119-121)
inline dg::LossBreakdown evaluate_losses(const dg::GraspObject& object, const dg::HandModel& hand,
                                         const dg::HandConfig& q, const dg::StabilityProtocol& protocol,
                                         const dg::SimParams& params) {
  if (static_cast<int>(q.joint_angles.size()) != hand.num_joints())
    throw std::runtime_error("hand: expected " + std::to_string(hand.num_joints()) + " joint angles, got " +
                             std::to_string(q.joint_angles.size()));
  return evaluate_losses(detail::thread_runtime(), detail::cached(object), detail::cached(hand), q, protocol,
                         params);
}

// dg::apply_gradient_step (losses.hpp:136; losses.cpp:92-102)
inline dg::HandConfig apply_gradient_step(const dg::HandConfig& q, const std::vector<double>& grad, double lr) {
  const int J = static_cast<int>(q.joint_angles.size());
  if (static_cast<int>(grad.size()) != 6 + J) throw std::runtime_error("gradient size mismatch");
  std::vector<double> qv = detail::pack(q), out(qv.size());
  detail::check(dgx_apply_gradient_step_joints(detail::thread_runtime().get(), J, 1, qv.data(), grad.data(), lr,
                                               out.data(), 0));
  return detail::unpack(out.data(), J);
}

// HandModel::forward(const HandConfig&) (hand.hpp:86) as a free function
inline std::vector<dg::Vec3> forward(const dg::HandModel& hand, const dg::HandConfig& q) {
  return forward(detail::thread_runtime(), detail::cached(hand), q);
}

}  // namespace dgx
