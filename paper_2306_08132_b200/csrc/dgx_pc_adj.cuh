// dgx_pc_adj.cuh — the lane adjoint as a producer / consumer pipeline
// (experimental: DGX_ADJ=pc). Included by dgx_kernels.cu after
// dgx_lane_adj.cuh, inside namespace dgx.
//
// The lane adjoint (one thread per (candidate, sim)) is latency-bound: a
// warp's per-position geometry is a long dependent FP64 chain and the batch
// gives it only ~6 warps per SM. The geometry of a position does not depend on
// the adjoint: it is a function of the frozen state of its run, which the
// forward's correction log already holds for every position. So here a CTA of
// 32 tasks has kPcProd producer warps that compute, block by block, each
// position's leak record (n = R g, the point p, c1 and k0 a with
// c0 = k0 a . G) into shared memory, tracking the log's run boundaries
// themselves, while one consumer warp walks the same positions applying the
// recurrence adj_x <- adj_x - s n, the emissions and the logged corrections
// (the only place the adjoint feeds back: G changes there, hence k0 a).
// One __syncthreads per block of kPcBlk positions, double-buffered records.
// Same closed forms as the lane adjoint; the R-node adjoint is accumulated in
// the world frame (sum rel (x) n s) and mapped back with R at corrections.
#pragma once

constexpr int kPcProd = 4;                 // producer warps per CTA
constexpr int kPcBlk = kPcProd * 2;        // positions per record block (2 per producer)
constexpr int kPcFields = 10;              // n 3, p 3, c1, k0 a 3
#ifndef DGX_PC_MINB
#define DGX_PC_MINB 3
#endif
__host__ __device__ inline int pc_smem_bytes() { return 2 * kPcBlk * kPcFields * 32 * 8; }

template <class Sdf>
__global__ void __launch_bounds__(32 * (kPcProd + 1), DGX_PC_MINB)
    pc_adj_kernel(const __grid_constant__ KHand H, const __grid_constant__ KObj O, const __grid_constant__ Sdf sdf,
                  const __grid_constant__ KSim S, const __grid_constant__ KOpt P, const __grid_constant__ KBuf buf,
                  int mode) {
  extern __shared__ __align__(16) unsigned char smem[];
  double* recs = reinterpret_cast<double*>(smem);  // [2][kPcBlk][kPcFields][32]
  const int M = S.M, N = H.N, L = H.L;
  const int lane = static_cast<int>(threadIdx.x & 31), warp = static_cast<int>(threadIdx.x >> 5);
  const bool consumer = warp == kPcProd;
  const size_t nt = static_cast<size_t>(buf.B) * M;
  const size_t t = static_cast<size_t>(blockIdx.x) * 32 + lane;
  const bool in = t < nt;
  const size_t tc = in ? t : nt - 1;
  const int b = static_cast<int>(tc / M), m = static_cast<int>(tc % M);
  const bool skip = !in || (mode == kModeOpt && P.k_begin > P.traj_k0 && buf.status[b] != kOk);
  double* ftT = buf.task_ft + tc;
  if (consumer && !skip)
    for (int c = 0; c < 6 * L; ++c) ftT[static_cast<size_t>(c) * nt] = 0.0;

  SimEnv e;
  e.lane = 0;
  e.N = N;
  e.gs = S.gs;
  const double* fkb = buf.fk + static_cast<size_t>(b) * (12 * L + 3 * N);
  e.px = fkb + 12 * L;
  e.py = fkb + 12 * L + N;
  e.pz = fkb + 12 * L + 2 * N;
  e.sample_link = H.sample_link;
  e.L = L;
  e.corr = buf.corr + tc * buf.cap_corr;
  e.slots = buf.slots + tc * buf.slot_stride;
  e.fric_order = buf.fric_order + tc * buf.slot_stride;
  e.cap_corr = buf.cap_corr;
  e.slot_cap = buf.slot_stride;
  e.O = &O;
  e.alpha = S.alpha;
  e.mu = S.mu;
  e.dt = S.dt;
  e.radius = S.radius;
  if (mode == kModeOpt) {
    const int k = P.k_begin;
    e.radius = P.iters > 1 ? P.r0 * (1.0 - static_cast<double>(k) / static_cast<double>(P.iters - 1)) : 0.0;
  }
  e.point_grads = buf.point_grads ? buf.point_grads + tc * N * 3 : nullptr;
  e.pts_global = 1;

  const FwdRec* rec = buf.fwd + tc;
  int status = rec->status;
  double residual = rec->residual;
  const double* vv = m < kMaxSims ? S.vel[m] : S.vel_dev + 3 * m;
  const V3 v_m{vv[0], vv[1], vv[2]};
  const V3 prev_x = O.com;
  const Q4 prev_q{1.0, 0.0, 0.0, 0.0};
  const V3 prev_thd{0.0, 0.0, 0.0};
  const V3 pred_xdot = v_m + V3{0.0 * e.dt, 0.0 * e.dt, 0.0 * e.dt};
  const V3 pred_x = prev_x + pred_xdot * e.dt;
  const Q4 pred_q = qnormalized(qmul(quat_exp(prev_thd * e.dt), prev_q));
  const int ncorr = rec->ncorr;
  const bool live = !skip && status == kOk && rec->touched != 0;
  V3 aX{0.0, 0.0, 0.0};
  Q4 aQ{0.0, 0.0, 0.0, 0.0};
  if (consumer && !skip && status == kOk) {
    const V3 x{rec->x[0], rec->x[1], rec->x[2]};
    const Q4 q{rec->q[0], rec->q[1], rec->q[2], rec->q[3]};
    const bool touched = rec->touched != 0;
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
    residual = n1 + n2;
    if (live) {
      const V3 a_xdot = n1 > 0.0 ? xdot / n1 : V3{0.0, 0.0, 0.0};
      const V3 a_thd = n2 > 0.0 ? thd / n2 : V3{0.0, 0.0, 0.0};
      aQ = qmul_adj_a(quat_log_adj(qd, a_thd * inv_dt), qconj(prev_q));
      aX = a_xdot * inv_dt;
      for (int j = rec->nfric - 1; j >= 0; --j) {
        SlotRec& s = e.slots[e.fric_order[j]];
        double a_lam = s.a_lam;
        V3 a_n{s.a_n[0], s.a_n[1], s.a_n[2]};
        friction_adj(e, prev_x, prev_q, s, aX, aQ, a_lam, a_n);
        s.a_lam = a_lam;
        s.a_n[0] = a_n.x; s.a_n[1] = a_n.y; s.a_n[2] = a_n.z;
      }
    }
  }
  // every warp of the CTA agrees on whether any task walks (a CTA-wide vote)
  const int any_live = __syncthreads_or(live ? 1 : 0);
  if (any_live) {
    const int top = S.gs * N - 1;
    const int nblk = (top + kPcBlk) / kPcBlk;  // blocks of kPcBlk positions, the last one partial
    auto slot = [&](int buf_i, int j, int f) -> double& {
      return recs[((static_cast<size_t>(buf_i) * kPcBlk + j) * kPcFields + f) * 32 + lane];
    };
    // state of the run a position belongs to (after correction kk; kk < 0: predicted)
    int kk = ncorr - 1;
    int f_k = live && kk >= 0 ? e.corr[kk].f : -1;
    V3 xk = pred_x;
    Q4 qk = pred_q;
    auto load_state = [&](int k2) {
      xk = pred_x;
      qk = pred_q;
      if (k2 >= 0) {
        const CorrRec& c = e.corr[k2];
        xk = V3{c.x[0], c.x[1], c.x[2]};
        qk = Q4{c.q[0], c.q[1], c.q[2], c.q[3]};
      }
    };
    if (live) load_state(kk);
    M3 Rk = rotation_matrix(qk);
    if (!consumer) {
      // ---- producer: 2 positions per block, this warp's slots 2 warp, 2 warp + 1
      for (int it = 0; it <= nblk; ++it) {
        if (it < nblk && live) {
#pragma unroll 1
          for (int u = 0; u < 2; ++u) {
            const int jb = 2 * warp + u;
            const int pos = top - kPcBlk * it - jb;
            if (pos < 0) break;
            // run boundaries at or above pos: the state of pos is after the last correction below it
            bool changed = false;
            while (kk >= 0 && f_k > pos) {
              --kk;
              f_k = kk >= 0 ? e.corr[kk].f : -1;
              changed = true;
            }
            if (changed) {
              load_state(kk);
              Rk = rotation_matrix(qk);
            }
            const int i = pos % N;
            const V3 p{e.px[i], e.py[i], e.pz[i]};
            double c1 = 0.0;
            V3 n{0.0, 0.0, 0.0}, k0a{0.0, 0.0, 0.0};
            if (!(kk >= 0 && f_k == pos)) {  // (a logged correction: the consumer reverses it)
              const V3 rel = p - xk;
              const V3 rl = ftmul_add(Rk, rel, e.O->com);
              GeoPre<Sdf> pre;
              pre.fetch(sdf, rl);
              FastEval fe = pre.finish(sdf, rl, e.radius);
              double sg = 1.0;
              bool on = fe.cls > 0;
              V3 g = fe.g;
              if (fe.cls == 0) {  // near the decision boundary: the exact (bit-exact) query decides
                PointEval pe;
                eval_point(sdf, e, i, xk, Rk, true, pe);
                on = !(pe.rho_d < 0.0);
                if (on) {
                  g = pe.q.grad;
                  sg = pe.fb ? static_cast<double>(pe.q.sign) : 1.0;
                }
              }
              if (on) {
                n = fmul(Rk, g);
                const V3 aa = fcross(rel, n);
                const V3 Ia = fmul(e.O->Iw, aa);
                const double w = e.O->inv_mass + fdot(aa, Ia);
                if (w >= 1e-12) {
                  const double lpc = rcp_fast(w);
                  c1 = e.alpha * e.O->inv_mass * lpc * sg;
                  k0a = aa * (0.5 * e.alpha * lpc * sg);
                } else {
                  n = V3{0.0, 0.0, 0.0};
                }
              }
            }
            const int bi = it & 1;
            slot(bi, jb, 0) = n.x; slot(bi, jb, 1) = n.y; slot(bi, jb, 2) = n.z;
            slot(bi, jb, 3) = p.x; slot(bi, jb, 4) = p.y; slot(bi, jb, 5) = p.z;
            slot(bi, jb, 6) = c1;
            slot(bi, jb, 7) = k0a.x; slot(bi, jb, 8) = k0a.y; slot(bi, jb, 9) = k0a.z;
          }
        }
        __syncthreads();
      }
    } else {
      // ---- consumer: the recurrence, emissions and logged corrections in order
      auto g_of = [&](Q4 qq, Q4 aq) {
        const V3 Hh{-qq.x * aq.w + qq.w * aq.x - qq.z * aq.y + qq.y * aq.z,
                    -qq.y * aq.w + qq.z * aq.x + qq.w * aq.y - qq.x * aq.z,
                    -qq.z * aq.w - qq.y * aq.x + qq.x * aq.y + qq.w * aq.z};
        return ftmul(e.O->Iw, Hh);
      };
      V3 G = g_of(qk, aQ);
      M3 aRw;  // sum rel (x) (n s) over the run: the R node's adjoint is aRw R
      for (int r = 0; r < 9; ++r) aRw.m[r] = 0.0;
      LaneFt acc;
      __syncthreads();  // block 0 produced
      for (int it = 1; it <= nblk; ++it) {
        const int bi = (it - 1) & 1;
        if (live) {
          for (int jb = 0; jb < kPcBlk; ++jb) {
            const int pos = top - kPcBlk * (it - 1) - jb;
            if (pos < 0) break;
            const int i = pos % N;
            if (pos == f_k) {  // this task's logged correction k (sim.hpp:215-245), reverse
              M3 aR;  // aRw R_k
              for (int r = 0; r < 3; ++r)
                for (int c = 0; c < 3; ++c)
                  aR.m[3 * r + c] = fma(aRw.m[3 * r + 2], Rk.m[6 + c],
                                        fma(aRw.m[3 * r + 1], Rk.m[3 + c], aRw.m[3 * r] * Rk.m[c]));
              aQ = qadd(aQ, rotmat_adj(qk, aR));
              const CorrRec& c = e.corr[kk];
              const SlotRec& sl = e.slots[c.slot];
              load_state(kk - 1);
              Rk = rotation_matrix(qk);
              bool ok = true;
              const CorrLin o = correction_linear(e, c, xk, qk, aX, aQ, sl.a_lam,
                                                  sl.last_corr == kk ? V3{sl.a_n[0], sl.a_n[1], sl.a_n[2]}
                                                                     : V3{0.0, 0.0, 0.0},
                                                  ok);
              if (!ok) status = kReplayMismatch;
              aX = o.aX;
              aQ = o.aQ;
              // the correction's R-node adjoint (state before it) in the world-frame accumulator
              for (int r = 0; r < 3; ++r)
                for (int cc = 0; cc < 3; ++cc)
                  aRw.m[3 * r + cc] = fma(o.aR.m[3 * r + 2], Rk.m[3 * cc + 2],
                                          fma(o.aR.m[3 * r + 1], Rk.m[3 * cc + 1], o.aR.m[3 * r] * Rk.m[3 * cc]));
              const V3 pp{e.px[i], e.py[i], e.pz[i]};
              double* d = ftT + static_cast<size_t>(6 * e.sample_link[i]) * nt;
              const V3 tq = cross(pp, o.a_rel);
              d[0] += o.a_rel.x; d[nt] += o.a_rel.y; d[2 * nt] += o.a_rel.z;
              d[3 * nt] += tq.x; d[4 * nt] += tq.y; d[5 * nt] += tq.z;
              add_point_grad(e, i, o.a_rel);
              --kk;
              f_k = kk >= 0 ? e.corr[kk].f : -1;
              G = g_of(qk, aQ);
              continue;
            }
            const V3 n{slot(bi, jb, 0), slot(bi, jb, 1), slot(bi, jb, 2)};
            const double c1 = slot(bi, jb, 6);
            const V3 k0a{slot(bi, jb, 7), slot(bi, jb, 8), slot(bi, jb, 9)};
            if (c1 != 0.0 || k0a.x != 0.0 || k0a.y != 0.0 || k0a.z != 0.0) {
              const V3 p{slot(bi, jb, 3), slot(bi, jb, 4), slot(bi, jb, 5)};
              const double s = fma(c1, fdot(n, aX), fdot(k0a, G));
              aX = fma3(-s, n, aX);
              const V3 a_rel = n * s;
              outer_acc(aRw, p - xk, a_rel);
              acc.add(ftT, nt, e.sample_link[i], a_rel, p);
              add_point_grad(e, i, a_rel);
            }
          }
        }
        __syncthreads();
      }
      if (live) {
        acc.flush(ftT, nt);
        if (S.discard) {
          l2_discard(e.corr, static_cast<size_t>(ncorr) * sizeof(CorrRec), 0, 1);
          l2_discard(e.slots, static_cast<size_t>(rec->nslot) * sizeof(SlotRec), 0, 1);
        }
      }
    }
  }
  if (!consumer || skip) return;
  buf.task_res[t] = residual;
  buf.task_stat[t] = status;
  if (buf.sim_res) buf.sim_res[t] = residual;
}
