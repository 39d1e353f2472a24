// dgx_drop.cu — batched scene drop: many independent rigid
// mesh objects falling onto the table plane z = 0, one warp per scene.
//
// Each step is the reference's step_on_table (sim.cpp:14-94) on values:
//   predict (sim.hpp:74-83) with gravity; world inverse inertia frozen at the
//   predicted orientation; gs_iters Gauss–Seidel sweeps over the mesh
//   vertices in index order, C = -z of the world vertex, correction along +z
//   with the angular update normalized(quat_exp(-lam I^-1 a) (x) theta) and R
//   recomputed; Coulomb friction over the activated vertices in index order;
//   velocities from the pose change when anything was corrected.
// The scene driver around it (run until at rest or a step cap)
// is specified but not implemented by the reference; here: stop once
// settle_steps consecutive steps made contact and left kinetic_energy
// (sim.cpp:8-12) below ke_tol (a single calm step also happens while a box
// balances on an edge), or at max_steps.
//
// Compiled with --fmad=false: every value rounds as in the reference, so a
// trajectory is bit-identical to step_on_table iterated on the CPU (parity
// mode P math for quat_exp / quat_log).
//
// Warp mapping: the 32 lanes test 32 consecutive vertices against the current
// pose (exact: the test is the reference's own arithmetic); the first violated
// vertex is corrected warp-uniformly and testing resumes right after it, which
// is the sequential sweep. Per-vertex contact slots (activated flag +
// accumulated lambda) live in a per-warp global scratch row and a shared
// bitmap, reset per step.
#include <cuda_runtime.h>

#include <cstdint>

#include "dgx_drop.cuh"

namespace dgx {

namespace {

constexpr unsigned kAll = 0xffffffffu;

struct Body {
  V3 x;
  Q4 q;
  V3 xd, w;
};

__device__ __forceinline__ double kinetic(const Body& s, const DropObj& O) {  // sim.cpp:8-12
  const M3 R = rotation_matrix(s.q);
  const M3 iw = mul(mul(R, O.Ibody), transposed(R));
  return 0.5 * O.mass * dot(s.xd, s.xd) + 0.5 * dot(s.w, mul(iw, s.w));
}

__device__ __forceinline__ V3 vtx(const DropObj& O, int i) {
  return V3{__ldg(O.verts + 3 * i), __ldg(O.verts + 3 * i + 1), __ldg(O.verts + 3 * i + 2)};
}

}  // namespace

__global__ void __launch_bounds__(128, 6) drop_kernel(const __grid_constant__ DropObj O, DropParams P, int B,
                                                   const double* __restrict__ in, double* __restrict__ out,
                                                   int* __restrict__ steps_out, double* __restrict__ ke_out,
                                                   double* __restrict__ stats_out, double* __restrict__ lam_all,
                                                   double* __restrict__ traj) {
  extern __shared__ unsigned drop_smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int nw = (O.V + 31) / 32;
  unsigned* bitmap = drop_smem + wib * nw;
  const int gw = blockIdx.x * (blockDim.x >> 5) + wib;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  double* lam = lam_all + static_cast<size_t>(gw) * O.V;
  const V3 zhat{0.0, 0.0, 1.0};
  const double inv_mass = 1.0 / O.mass;
  const double inv_dt = 1.0 / P.dt;

  for (int b = gw; b < B; b += nwarps) {
    const double* si = in + 13 * static_cast<size_t>(b);
    Body s{V3{si[0], si[1], si[2]}, Q4{si[3], si[4], si[5], si[6]}, V3{si[7], si[8], si[9]},
           V3{si[10], si[11], si[12]}};
    int steps = 0, calm = 0;
    double ke = kinetic(s, O);
    int n_corr = 0, n_active = 0, n_sing = 0;
    double max_pen = 0.0;
    for (int k = 0; k < P.max_steps; ++k) {
      // ---- predict (sim.hpp:74-83)
      const Body prev = s;
      Body st = s;
      st.xd = prev.xd + V3{P.gravity.x * P.dt, P.gravity.y * P.dt, P.gravity.z * P.dt};
      st.x = prev.x + P.dt * st.xd;
      st.q = qnormalized(qmul(quat_exp(P.dt * prev.w), prev.q));
      st.w = prev.w;
      // world inertia inverse at the predicted orientation (sim_detail::world_inertia_inv)
      const M3 Rp = rotation_matrix(st.q);
      const M3 iw_inv = mul(mul(Rp, O.Iinv), transposed(Rp));
      bool touched = false;
      for (int wd = lane; wd < nw; wd += 32) bitmap[wd] = 0u;
      __syncwarp();
      // ---- Gauss-Seidel over vertices (sim.cpp:30-54)
      M3 R = rotation_matrix(st.q);
      for (int sweep = 0; sweep < P.gs; ++sweep) {
        R = rotation_matrix(st.q);
        int pos = 0;
        while (pos < O.V) {
          const int i = pos + lane;
          bool viol = false;
          if (i < O.V) {
            const V3 wv = st.x + mul(R, vtx(O, i) - O.com);
            viol = -wv.z > 0.0;
          }
          const unsigned m = __ballot_sync(kAll, viol);
          if (m == 0u) {
            pos += 32;
            continue;
          }
          const int j = pos + __ffs(m) - 1;
          // warp-uniform correction of vertex j (every lane computes the same values)
          const V3 wv = st.x + mul(R, vtx(O, j) - O.com);
          const double C = -wv.z;
          const V3 arm = wv - st.x;
          const V3 a = -cross(arm, zhat);
          const V3 iwa = mul(iw_inv, a);
          const double w_eff = inv_mass + dot(a, iwa);
          if (w_eff < 1e-12) {
            ++n_sing;
          } else {
            const double lm = C / w_eff;
            st.x = st.x + (inv_mass * lm) * zhat;
            st.q = qnormalized(qmul(quat_exp(-lm * iwa), st.q));
            R = rotation_matrix(st.q);
            touched = true;
            if (lane == 0) {
              const unsigned bit = 1u << (j & 31);
              if (!(bitmap[j >> 5] & bit)) {
                bitmap[j >> 5] |= bit;
                lam[j] = 0.0;
                ++n_active;
              }
              lam[j] += lm;
            }
            ++n_corr;
          }
          __syncwarp();
          pos = j + 1;
        }
      }
      // ---- friction over activated vertices in index order (sim.cpp:56-78)
      if (P.mu > 0.0) {
        for (int wd = 0; wd < nw; ++wd) {
          unsigned bits = bitmap[wd];
          while (bits) {
            const int i = wd * 32 + __ffs(bits) - 1;
            bits &= bits - 1u;
            const double lambda_n = lam[i];
            if (lambda_n <= 0.0) continue;
            const V3 rb = vtx(O, i) - O.com;
            const V3 before = prev.x + rotate(prev.q, rb);
            const V3 arm = rotate(st.q, rb);
            const V3 after = st.x + arm;
            const V3 u = after - before;
            const V3 u_t{u.x, u.y, 0.0};
            const double ut = norm(u_t);
            if (ut < 1e-12) continue;
            const V3 t = u_t / ut;
            const V3 at = cross(arm, t);
            const V3 iwat = mul(iw_inv, at);
            const double w_t = inv_mass + dot(at, iwat);
            if (w_t < 1e-12) continue;
            const double a1 = ut / w_t, a2 = P.mu * lambda_n;
            const double lam_t = a2 < a1 ? a2 : a1;  // std::min(a1, a2)
            st.x = st.x - (inv_mass * lam_t) * t;
            st.q = qnormalized(qmul(quat_exp(-lam_t * iwat), st.q));
            touched = true;
            ++n_corr;
          }
        }
      }
      // ---- velocities (sim.cpp:80-84)
      if (touched) {
        st.xd = (st.x - prev.x) * inv_dt;
        st.w = quat_log(qmul(st.q, qconj(prev.q))) * inv_dt;
      }
      s = st;
      steps = k + 1;
      if (P.measure) {  // sim.cpp:86-92
        const M3 Rf = rotation_matrix(s.q);
        double mp = 0.0;
        for (int i = lane; i < O.V; i += 32) {
          const double z = (s.x + mul(Rf, vtx(O, i) - O.com)).z;
          if (z < 0.0) mp = mp < -z ? -z : mp;
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double v = __shfl_xor_sync(kAll, mp, o);
          mp = mp < v ? v : mp;
        }
        max_pen = max_pen < mp ? mp : max_pen;
      }
      if (traj && P.record_every > 0 && (k + 1) % P.record_every == 0 && lane < 13) {
        const double v[13] = {s.x.x, s.x.y, s.x.z, s.q.w, s.q.x, s.q.y, s.q.z, s.xd.x, s.xd.y, s.xd.z,
                              s.w.x, s.w.y, s.w.z};
        const int rows = P.max_steps / P.record_every;
        traj[(static_cast<size_t>(b) * rows + (k + 1) / P.record_every - 1) * 13 + lane] = v[lane];
      }
      ke = kinetic(s, O);
      calm = (touched && ke < P.ke_tol) ? calm + 1 : 0;
      if (calm >= P.settle_steps && k + 1 >= P.min_steps) break;
    }
    if (lane == 0) {
      double* so = out + 13 * static_cast<size_t>(b);
      so[0] = s.x.x; so[1] = s.x.y; so[2] = s.x.z;
      so[3] = s.q.w; so[4] = s.q.x; so[5] = s.q.y; so[6] = s.q.z;
      so[7] = s.xd.x; so[8] = s.xd.y; so[9] = s.xd.z;
      so[10] = s.w.x; so[11] = s.w.y; so[12] = s.w.z;
      steps_out[b] = steps;
      ke_out[b] = ke;
      if (stats_out) {
        double* st = stats_out + 4 * static_cast<size_t>(b);
        st[0] = n_active; st[1] = n_corr; st[2] = n_sing; st[3] = max_pen;
      }
    }
    __syncwarp();
  }
}

cudaError_t launch_drop(const DropObj& O, const DropParams& P, int B, const double* in, double* out, int* steps,
                        double* ke, double* stats, double* lam_scratch, int warps_total, double* traj,
                        cudaStream_t st) {
  if (B <= 0) return cudaSuccess;
  const int wpb = 4;
  const int blocks = (warps_total + wpb - 1) / wpb;
  const size_t smem = static_cast<size_t>(wpb) * ((O.V + 31) / 32) * sizeof(unsigned);
  drop_kernel<<<blocks, 32 * wpb, smem, st>>>(O, P, B, in, out, steps, ke, stats, lam_scratch, traj);
  return cudaGetLastError();
}

}  // namespace dgx
