// dgx_drop.cuh — batched scene drop (step_on_table, sim.cpp:14-94).
#pragma once

#include <cuda_runtime.h>

#include "dgx_geom.h"

namespace dgx {

struct DropObj {
  const double* verts;  // [V,3] canonical-frame mesh vertices (the contact samples, sim.cpp:28)
  int V;
  double mass;
  V3 com;
  M3 Ibody, Iinv;       // InertialData::inertia_body / inertia_body_inv
};

struct DropParams {
  double dt, mu;
  int gs;
  V3 gravity;
  int max_steps, min_steps;
  double ke_tol;
  int record_every;  // > 0 with traj: state every record_every steps
  int settle_steps;  // consecutive calm contact steps that end a drop
  int measure;       // SolveStats::measure_residual (max table penetration over steps)
};

// in/out [B,13] RigidState rows: x(3), theta w,x,y,z (4), xdot(3), thetadot(3);
// steps [B]; ke [B] final kinetic energy; stats [B,4] (active contacts,
// corrections, singular skipped, max penetration) accumulated over the steps
// as one SolveStats; lam_scratch [warps_total, V]
cudaError_t launch_drop(const DropObj& O, const DropParams& P, int B, const double* in, double* out, int* steps,
                        double* ke, double* stats, double* lam_scratch, int warps_total, double* traj,
                        cudaStream_t st);

}  // namespace dgx
