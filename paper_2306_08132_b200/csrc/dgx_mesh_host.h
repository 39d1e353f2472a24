// dgx_mesh_host.h — host-side mesh preparation for the MeshSdf backend.
#pragma once

#include <cstdint>
#include <vector>

#include "dgx_mesh.h"

namespace dgx {

struct MeshHost {
  std::vector<MeshNode> nodes;  // DFS preorder, root 0 (bvh.cpp:66-103)
  std::vector<MeshFace> faces;  // leaf order
  std::vector<int> tri;         // [F,3]
  std::vector<double> vx, vn;   // [V,3]
  std::vector<int> vf_off, vf_idx;  // vertex -> incident faces (CSR)
  double blo[3], bhi[3];
  int depth = 0;
};

// TriMesh::finalize (mesh.cpp:12-71) validation + area-weighted vertex normals
// (or the given unit normals, as TriMesh::set_vertex_normals, mesh.cpp:73-81),
// then Bvh::build (bvh.cpp:148-163). Throws std::runtime_error with the
// reference's messages.
void mesh_prepare(int nv, const double* V, int nf, const int32_t* F, const double* VN, MeshHost& out);

// inertia_from_mesh (rigid.cpp:24-94); mesh validated as above.
void mesh_inertia(int nv, const double* V, int nf, const int32_t* F, double density, double& mass, double* com,
                  double* I, double* Iinv);

// fixed ray directions of Bvh::sign_at (bvh.cpp:143-144, 250) and 1/dir
void mesh_ray_dirs(double dir[3][3], double inv[3][3]);

}  // namespace dgx
