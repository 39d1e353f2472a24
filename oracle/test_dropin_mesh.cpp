// oracle/test_dropin_mesh.cpp — TEST INFRASTRUCTURE: the drop-in C++ API
// (include/dgx/diffgrasp.hpp) on the reference's OWN mesh object. Linked with
// the unmodified reference objects including its real losses.cpp (no shim),
// in parity mode P (shared sin/cos/atan2). A dg::GraspObject built by the
// reference (make_icosphere, MeshSdf, inertia_from_mesh) is handed to
// dgx::Object unchanged; dgx::loss_gradient / evaluate_losses /
// dilated / dilated_within are compared with dg::loss_gradient /
// dg::evaluate_losses / MeshSdf::dilated / MeshSdf::dilated_within.
// Prints "DROPIN MESH OK" and exits 0 on success.
#include <cmath>
#include <cstdio>
#include <vector>

#include "diffgrasp/assets.hpp"
#include "dgx/diffgrasp.hpp"

static int failures = 0;
#define EXPECT(c, ...) do { if (!(c)) { ++failures; std::printf("FAIL %s:%d: ", __FILE__, __LINE__); std::printf(__VA_ARGS__); std::printf("\n"); } } while (0)

int main() {
  dg::HandModel hand = dg::make_three_finger_hand(2000, 12345);
  dg::GraspObject go(dg::make_icosphere(0.025, 3), 1000.0, 0.75);
  dgx::Runtime rt(0);
  dgx::Hand dh(rt, hand);
  dgx::Object mobj(rt, go);
  dg::StabilityProtocol proto = dg::StabilityProtocol::standard();
  std::vector<dg::HandConfig> qs;
  for (int b = 0; b < 4; ++b) {
    dg::HandConfig q = hand.mid_range_config();
    q.base_position = {0.001 * b, -0.0005 * b, -0.040 + 0.0007 * b};
    qs.push_back(q);
  }
  int contacts = 0;
  for (double radius : {0.0, 0.01}) {
    dg::SimParams sp;
    sp.dilation_radius = radius;
    auto batch = dgx::loss_gradient(rt, mobj, dh, std::span<const dg::HandConfig>(qs), proto, sp);
    for (std::size_t b = 0; b < qs.size(); ++b) {
      dg::LossGradient ref = dg::loss_gradient(go, hand, qs[b], proto, sp);
      EXPECT(batch[b].losses.stable == ref.losses.stable && batch[b].losses.qrange == ref.losses.qrange &&
                 batch[b].losses.qlimit == ref.losses.qlimit,
             "losses differ b=%zu r=%g: %.17g vs %.17g", b, radius, batch[b].losses.stable, ref.losses.stable);
      double mx = 0, err = 0;
      for (std::size_t i = 0; i < ref.d_stable.size(); ++i) {
        mx = std::fmax(mx, std::fabs(ref.d_stable[i]));
        err = std::fmax(err, std::fabs(batch[b].d_stable[i] - ref.d_stable[i]));
      }
      EXPECT(err <= 1e-9 * mx, "gradient rel err %.3e", mx > 0 ? err / mx : err);
      contacts += mx > 0;
      dg::LossBreakdown ev = dgx::evaluate_losses(rt, mobj, dh, qs[b], proto, sp);
      dg::LossBreakdown er = dg::evaluate_losses(go, hand, qs[b], proto, sp);
      EXPECT(ev.stable == er.stable && ev.qrange == er.qrange && ev.qlimit == er.qlimit, "evaluate_losses differs");
    }
  }
  EXPECT(contacts > 0, "no case produced a nonzero gradient");
  std::vector<dg::Vec3> pts = {{0.03, 0.001, 0.002}, {0.0, 0.0, 0.0}, {0.0249, 0.0, 0.0}, {0.1, 0.1, 0.1},
                               {0.0, 0.026, 0.001}, {-0.02, 0.01, 0.012}};
  for (const auto& r : pts) {
    for (double radius : {0.0, 0.002}) {
      dg::PhongQuery a = dgx::dilated(rt, mobj, r, radius);
      dg::PhongQuery b = go.sdf.dilated(r, radius);
      EXPECT(a.rho == b.rho && a.sign == b.sign && a.grad.x == b.grad.x && a.grad.y == b.grad.y &&
                 a.grad.z == b.grad.z && a.smoothed_point.x == b.smoothed_point.x &&
                 a.smoothed_point.y == b.smoothed_point.y && a.smoothed_point.z == b.smoothed_point.z,
             "dilated differs: %.17g vs %.17g", a.rho, b.rho);
      auto aw = dgx::dilated_within(rt, mobj, r, radius);
      auto bw = go.sdf.dilated_within(r, radius, 0.005);
      EXPECT(aw.has_value() == bw.has_value() && (!aw || aw->rho == bw->rho), "dilated_within differs");
    }
  }
  // ---- the reference's own signatures, call sites unchanged but for the
  // namespace (dg:: -> dgx::): standard protocol, T = 2 steps, M = 9 velocities
  dg::StabilityProtocol t2 = dg::StabilityProtocol::standard(0.5, 2);
  dg::StabilityProtocol m9 = dg::StabilityProtocol::standard();
  m9.velocities.push_back({0.3, 0.3, 0.0});
  m9.velocities.push_back({0.0, 0.2, -0.4});
  dg::GraspObject cube(dg::make_box(0.04, 0.04, 0.04), 1000.0, 0.75);
  int nonzero = 0;
  for (const dg::GraspObject* obj : {&go, &cube, &go}) {  // two objects through the per-thread upload cache
    for (const dg::StabilityProtocol* pr : {&proto, &t2, &m9}) {
      dg::SimParams sp;
      sp.dilation_radius = 0.01;
      for (std::size_t b = 0; b < qs.size(); ++b) {
        dg::LossGradient a = dgx::loss_gradient(*obj, hand, qs[b], *pr, sp);
        dg::LossGradient r = dg::loss_gradient(*obj, hand, qs[b], *pr, sp);
        EXPECT(a.losses.stable == r.losses.stable && a.losses.qrange == r.losses.qrange &&
                   a.losses.qlimit == r.losses.qlimit,
               "ref-signature losses differ (M=%d T=%d b=%zu): %.17g vs %.17g", pr->m(), pr->steps, b,
               a.losses.stable, r.losses.stable);
        double mx = 0, err = 0;
        for (std::size_t i = 0; i < r.d_stable.size(); ++i) {
          mx = std::fmax(mx, std::fabs(r.d_stable[i]));
          err = std::fmax(err, std::fabs(a.d_stable[i] - r.d_stable[i]));
        }
        EXPECT(err <= 1e-8 * mx, "ref-signature gradient rel err %.3e (M=%d T=%d)", mx > 0 ? err / mx : err, pr->m(),
               pr->steps);
        nonzero += mx > 0;
        dg::LossBreakdown ea = dgx::evaluate_losses(*obj, hand, qs[b], *pr, sp);
        dg::LossBreakdown er = dg::evaluate_losses(*obj, hand, qs[b], *pr, sp);
        EXPECT(ea.stable == er.stable && ea.qrange == er.qrange && ea.qlimit == er.qlimit,
               "ref-signature evaluate_losses differs (M=%d T=%d)", pr->m(), pr->steps);
      }
    }
  }
  EXPECT(nonzero > 0, "no reference-signature case produced a gradient");
  {
    auto g = dg::loss_gradient(go, hand, qs[1], proto, dg::SimParams{}).weighted(dg::LossWeights{});
    for (double& x : g) x = std::tanh(x);
    dg::HandConfig a = dgx::apply_gradient_step(qs[1], g, 1e-3);
    dg::HandConfig r = dg::apply_gradient_step(qs[1], g, 1e-3);
    EXPECT(a.base_position.x == r.base_position.x && a.base_position.z == r.base_position.z &&
               a.base_orientation.w == r.base_orientation.w && a.base_orientation.y == r.base_orientation.y &&
               a.joint_angles == r.joint_angles,
           "ref-signature apply_gradient_step differs");
    auto pa = dgx::forward(hand, qs[2]);
    auto pb = hand.forward(qs[2]);
    bool same = pa.size() == pb.size();
    for (std::size_t i = 0; same && i < pa.size(); ++i) same = pa[i].x == pb[i].x && pa[i].y == pb[i].y && pa[i].z == pb[i].z;
    EXPECT(same, "ref-signature forward differs");
  }
  if (failures == 0) std::printf("DROPIN MESH OK\n");
  return failures == 0 ? 0 : 1;
}
