// oracle/test_dropin.cpp — TEST INFRASTRUCTURE: exercises the drop-in C++ API
// (include/dgx/diffgrasp.hpp) exactly as a user of the reference library would
// (dg::HandModel, dg::HandConfig, dg::StabilityProtocol, dg::SimParams in;
// dg::LossGradient / dg::LossBreakdown / dg::HandConfig out) and checks it
// against the reference itself (parity mode P build, linked in-process).
// Prints "DROPIN OK" and exits 0 on success.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "diffgrasp/assets.hpp"
#include "dgx/diffgrasp.hpp"

extern "C" {  // reference loss_gradient with the analytic sphere (oracle/ref_shim.cpp)
void* dgr_object_icosphere(double radius, int subdiv, double density, double alpha);
void dgr_object_use_sphere(void* o, double cx, double cy, double cz, double r);
void dgr_object_set_inertial(void* o, double mass, const double* com, const double* I, const double* Iinv);
struct Params { double dt, mu; int gs_iters, steps; double dilation_radius, alpha_leak, speed, w_stable, w_qrange, w_qlimit; };
int dgr_loss_gradient(void* o, void* hp, const double* q, const Params* p, double* losses, double* ds, double* dr,
                      double* dl);
int dgr_evaluate_losses(void* o, void* hp, const double* q, const Params* p, double* losses);
}

static int failures = 0;
#define EXPECT(c, ...) do { if (!(c)) { ++failures; std::printf("FAIL %s:%d: ", __FILE__, __LINE__); std::printf(__VA_ARGS__); std::printf("\n"); } } while (0)

int main() {
  dg::HandModel hand = dg::make_three_finger_hand(2000, 12345);
  const double R = 0.025, rho = 1000.0;
  const double mass = rho * 4.0 / 3.0 * M_PI * R * R * R, I = 0.4 * mass * R * R;
  dg::InertialData in;
  in.mass = mass;
  in.com = {0, 0, 0};
  in.inertia_body = dg::Mat3::identity();
  in.inertia_body_inv = dg::Mat3::identity();
  for (int k : {0, 4, 8}) { in.inertia_body.m[k] = I; in.inertia_body_inv.m[k] = 1.0 / I; }

  dgx::Runtime rt(0);
  dgx::Hand dh(rt, hand);
  dgx::SdfSpec spec;
  spec.kind = DGX_SDF_SPHERE;
  spec.radius = R;
  dgx::Object dobj(rt, spec, in);

  void* ro = dgr_object_icosphere(0.02, 1, 1000.0, 0.75);
  dgr_object_use_sphere(ro, 0, 0, 0, R);
  double com[3] = {0, 0, 0};
  dgr_object_set_inertial(ro, mass, com, in.inertia_body.m.data(), in.inertia_body_inv.m.data());

  dg::StabilityProtocol proto = dg::StabilityProtocol::standard();
  std::vector<dg::HandConfig> qs;
  for (int b = 0; b < 4; ++b) {
    dg::HandConfig q = hand.mid_range_config();
    q.base_position = {0.001 * b, -0.0005 * b, -0.040 + 0.0007 * b};
    qs.push_back(q);
  }
  // forward: bit-exact with HandModel::forward
  for (const auto& q : qs) {
    auto a = dgx::forward(rt, dh, q);
    auto b = hand.forward(q);
    bool same = a.size() == b.size();
    for (std::size_t i = 0; same && i < a.size(); ++i) same = a[i].x == b[i].x && a[i].y == b[i].y && a[i].z == b[i].z;
    EXPECT(same, "forward differs");
  }
  for (double radius : {0.0, 0.01}) {
    dg::SimParams sp;
    sp.dilation_radius = radius;
    Params p{sp.dt, sp.mu, sp.gs_iters, proto.steps, radius, sp.leak.alpha_leak, 0.5, 1.0, 0.01, 1.0};
    auto batch = dgx::loss_gradient(rt, dobj, dh, std::span<const dg::HandConfig>(qs), proto, sp);
    for (std::size_t b = 0; b < qs.size(); ++b) {
      std::vector<double> qv = dgx::detail::pack(qs[b]);
      const int D = 6 + hand.num_joints();
      double l[3];
      std::vector<double> ds(D), dr(D), dl(D);
      dgr_loss_gradient(ro, &hand, qv.data(), &p, l, ds.data(), dr.data(), dl.data());
      EXPECT(batch[b].losses.stable == l[0] && batch[b].losses.qrange == l[1] && batch[b].losses.qlimit == l[2],
             "losses differ b=%zu: %.17g vs %.17g", b, batch[b].losses.stable, l[0]);
      double mx = 0, err = 0;
      for (int i = 0; i < D; ++i) {
        mx = std::fmax(mx, std::fabs(ds[i]));
        err = std::fmax(err, std::fabs(batch[b].d_stable[i] - ds[i]));
      }
      EXPECT(err <= 1e-9 * mx, "gradient rel err %.3e", mx > 0 ? err / mx : err);
      dg::LossGradient one = dgx::loss_gradient(rt, dobj, dh, qs[b], proto, sp);
      EXPECT(one.losses.stable == batch[b].losses.stable, "batch-of-one differs");
      dg::LossBreakdown ev = dgx::evaluate_losses(rt, dobj, dh, qs[b], proto, sp);
      double le[3];
      dgr_evaluate_losses(ro, &hand, qv.data(), &p, le);
      EXPECT(ev.stable == le[0] && ev.qrange == le[1] && ev.qlimit == le[2], "evaluate_losses differs");
      // apply_gradient_step: bit-exact with the reference
      auto g = one.weighted(dg::LossWeights{});
      for (double& x : g) x = std::tanh(x);  // keep the step O(lr)
      dg::HandConfig a = dgx::apply_gradient_step(rt, dh, qs[b], g, 1e-3);
      dg::HandConfig r = dg::apply_gradient_step(qs[b], g, 1e-3);
      bool same = a.base_position.x == r.base_position.x && a.base_orientation.w == r.base_orientation.w &&
                  a.base_orientation.z == r.base_orientation.z && a.joint_angles == r.joint_angles;
      EXPECT(same, "apply_gradient_step differs");
    }
  }
  // error behaviour: negative dilation -> std::invalid_argument (sdf.cpp:84)
  try {
    dg::SimParams bad;
    bad.dilation_radius = -0.1;
    dgx::loss_gradient(rt, dobj, dh, qs[0], proto, bad);
    EXPECT(false, "no exception for negative dilation");
  } catch (const std::invalid_argument&) {
  }
  // optimize runs and keeps unit quaternions
  auto fin = dgx::optimize(rt, dobj, dh, std::span<const dg::HandConfig>(qs), proto, dg::SimParams{}, dg::LossWeights{},
                           dgx::OptimizeConfig{20});
  for (const auto& q : fin) {
    const auto& o = q.base_orientation;
    EXPECT(std::fabs(o.w * o.w + o.x * o.x + o.y * o.y + o.z * o.z - 1.0) < 1e-12, "non-unit quaternion");
  }
  if (failures == 0) std::printf("DROPIN OK\n");
  return failures == 0 ? 0 : 1;
}
