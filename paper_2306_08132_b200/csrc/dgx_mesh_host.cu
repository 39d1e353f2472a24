// dgx_mesh_host.cu — host-only: mesh validation, vertex normals, the BVH and
// mass properties, each following the reference routine cited per function.
// Host code without FMA contraction (x86-64 baseline ISA has no FMA), so
// values round as in the reference build.
#include "dgx_mesh_host.h"

#include <algorithm>
#include <cmath>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>
#include <utility>

namespace dgx {

namespace {

struct Mesh {
  int nv, nf;
  const double* V;
  const int32_t* F;
  V3 v(int f, int k) const {
    const double* p = V + 3 * F[3 * f + k];
    return V3{p[0], p[1], p[2]};
  }
};

struct Box {
  double lo[3] = {1e300, 1e300, 1e300};
  double hi[3] = {-1e300, -1e300, -1e300};
  void expand(V3 p) {  // Box3::expand (vec.hpp:194-197), std::min / std::max
    const double a[3] = {p.x, p.y, p.z};
    for (int i = 0; i < 3; ++i) {
      lo[i] = a[i] < lo[i] ? a[i] : lo[i];
      hi[i] = hi[i] < a[i] ? a[i] : hi[i];
    }
  }
};

// mesh.cpp:12-58 checks + area-weighted normals (mesh.cpp:60-70)
void validate(const Mesh& m, std::vector<double>& vn_out, bool want_normals) {
  std::vector<V3> fn(m.nf);
  std::vector<double> area(m.nf);
  for (int f = 0; f < m.nf; ++f) {
    for (int k = 0; k < 3; ++k) {
      const int idx = m.F[3 * f + k];
      if (idx < 0 || idx >= m.nv)
        throw std::runtime_error("mesh: face " + std::to_string(f) + " references vertex " + std::to_string(idx) +
                                 " out of range");
    }
    const V3 n = cross(m.v(f, 1) - m.v(f, 0), m.v(f, 2) - m.v(f, 0));
    const double a2 = norm(n);
    if (a2 <= 1e-16) throw std::runtime_error("mesh: degenerate (zero area) face " + std::to_string(f));
    fn[f] = n / a2;
    area[f] = 0.5 * a2;
  }
  std::map<std::pair<int, int>, int> directed;
  for (int f = 0; f < m.nf; ++f) {
    for (int k = 0; k < 3; ++k) {
      const int a = m.F[3 * f + k], b = m.F[3 * f + (k + 1) % 3];
      if (a == b)
        throw std::runtime_error("mesh: face " + std::to_string(f) + " repeats vertex " + std::to_string(a));
      auto ins = directed.emplace(std::make_pair(a, b), f);
      if (!ins.second)
        throw std::runtime_error("mesh: not watertight, directed edge (" + std::to_string(a) + "," +
                                 std::to_string(b) + ") shared by faces " + std::to_string(ins.first->second) +
                                 " and " + std::to_string(f));
    }
  }
  for (const auto& kv : directed) {
    if (!directed.count({kv.first.second, kv.first.first}))
      throw std::runtime_error("mesh: not watertight, edge (" + std::to_string(kv.first.first) + "," +
                               std::to_string(kv.first.second) + ") of face " + std::to_string(kv.second) +
                               " has no opposite");
  }
  double vol = 0.0;  // TriMesh::signed_volume (mesh.cpp:83-88)
  for (int f = 0; f < m.nf; ++f) vol += dot(m.v(f, 0), cross(m.v(f, 1), m.v(f, 2))) / 6.0;
  if (vol <= 0.0) throw std::runtime_error("mesh: inconsistent winding, signed volume is not positive");
  if (!want_normals) return;
  std::vector<V3> acc(m.nv, V3{0.0, 0.0, 0.0});
  for (int f = 0; f < m.nf; ++f) {
    const V3 w = area[f] * fn[f];
    for (int k = 0; k < 3; ++k) {
      V3& t = acc[m.F[3 * f + k]];
      t = t + w;
    }
  }
  vn_out.resize(3 * static_cast<size_t>(m.nv));
  for (int i = 0; i < m.nv; ++i) {
    const double n = norm(acc[i]);
    if (n <= 1e-16) throw std::runtime_error("mesh: vertex " + std::to_string(i) + " has zero normal");
    const V3 u = acc[i] / n;
    vn_out[3 * i] = u.x; vn_out[3 * i + 1] = u.y; vn_out[3 * i + 2] = u.z;
  }
}

// Bvh build_node (bvh.cpp:66-103). The children's face SETS are the lower /
// upper count/2 faces under the total order (centroid[axis], face id), so a
// sort yields the same partition as the reference's nth_element; node ids are
// assigned in the same DFS preorder.
struct Builder {
  const Mesh& m;
  std::vector<V3> cen;
  std::vector<int> order;
  std::vector<MeshNode>& nodes;
  int depth = 0;

  int build(int first, int count, int level) {
    depth = std::max(depth, level);
    const int id = static_cast<int>(nodes.size());
    nodes.push_back(MeshNode{});
    Box box;
    for (int i = first; i < first + count; ++i) {
      const int f = order[i];
      box.expand(m.v(f, 0));
      box.expand(m.v(f, 1));
      box.expand(m.v(f, 2));
    }
    for (int k = 0; k < 3; ++k) {
      nodes[id].lo[k] = box.lo[k];
      nodes[id].hi[k] = box.hi[k];
    }
    if (count <= 4) {
      nodes[id].left = nodes[id].right = -1;
      nodes[id].first = first;
      nodes[id].count = count;
      return id;
    }
    Box cb;
    for (int i = first; i < first + count; ++i) cb.expand(cen[order[i]]);
    const double ext[3] = {cb.hi[0] - cb.lo[0], cb.hi[1] - cb.lo[1], cb.hi[2] - cb.lo[2]};
    int axis = 0;
    if (ext[1] > ext[0]) axis = 1;
    if (ext[2] > ext[axis]) axis = 2;
    auto key = [&](int f) {
      const V3& c = cen[f];
      return axis == 0 ? c.x : (axis == 1 ? c.y : c.z);
    };
    std::sort(order.begin() + first, order.begin() + first + count, [&](int fa, int fb) {
      const double ca = key(fa), cb2 = key(fb);
      if (ca != cb2) return ca < cb2;
      return fa < fb;
    });
    const int mid = first + count / 2;
    const int left = build(first, mid - first, level + 1);
    const int right = build(mid, first + count - mid, level + 1);
    nodes[id].left = left;
    nodes[id].right = right;
    nodes[id].first = 0;
    nodes[id].count = 0;
    return id;
  }
};

}  // namespace

void mesh_prepare(int nv, const double* V, int nf, const int32_t* F, const double* VN, MeshHost& out) {
  if (nv < 4 || nf < 4 || !V || !F) throw std::runtime_error("mesh: needs >= 4 vertices and >= 4 faces");
  const Mesh m{nv, nf, V, F};
  validate(m, out.vn, VN == nullptr);
  if (VN) {  // TriMesh::set_vertex_normals (mesh.cpp:73-81)
    for (int i = 0; i < nv; ++i) {
      const double n = norm(V3{VN[3 * i], VN[3 * i + 1], VN[3 * i + 2]});
      if (std::abs(n - 1.0) > 1e-9)
        throw std::runtime_error("mesh: normal " + std::to_string(i) + " is not unit length");
    }
    out.vn.assign(VN, VN + 3 * static_cast<size_t>(nv));
  }
  out.vx.assign(V, V + 3 * static_cast<size_t>(nv));
  out.tri.assign(F, F + 3 * static_cast<size_t>(nf));
  Box b;
  for (int i = 0; i < nv; ++i) b.expand(V3{V[3 * i], V[3 * i + 1], V[3 * i + 2]});
  for (int k = 0; k < 3; ++k) {
    out.blo[k] = b.lo[k];
    out.bhi[k] = b.hi[k];
  }
  Builder bd{m, std::vector<V3>(nf), std::vector<int>(nf), out.nodes};
  out.nodes.clear();
  out.nodes.reserve(2 * static_cast<size_t>(nf));
  for (int f = 0; f < nf; ++f) {
    bd.order[f] = f;
    bd.cen[f] = (m.v(f, 0) + m.v(f, 1) + m.v(f, 2)) / 3.0;
  }
  bd.build(0, nf, 0);
  out.depth = bd.depth;
  if (out.depth + 2 > kMeshStack) throw std::runtime_error("mesh: BVH too deep for the device traversal stack");
  out.vf_off.assign(nv + 1, 0);
  for (int i = 0; i < 3 * nf; ++i) ++out.vf_off[F[i] + 1];
  for (int v = 0; v < nv; ++v) out.vf_off[v + 1] += out.vf_off[v];
  out.vf_idx.assign(3 * static_cast<size_t>(nf), 0);
  {
    std::vector<int> fill(out.vf_off.begin(), out.vf_off.end() - 1);
    for (int f = 0; f < nf; ++f)
      for (int k = 0; k < 3; ++k) out.vf_idx[fill[F[3 * f + k]]++] = f;
  }
  out.faces.resize(nf);
  for (int i = 0; i < nf; ++i) {
    const int f = bd.order[i];
    MeshFace& r = out.faces[i];
    for (int k = 0; k < 3; ++k) {
      r.a[k] = V[3 * F[3 * f] + k];
      r.b[k] = V[3 * F[3 * f + 1] + k];
      r.c[k] = V[3 * F[3 * f + 2] + k];
    }
    r.f = f;
    r.pad = 0;
  }
}

void mesh_ray_dirs(double dir[3][3], double inv[3][3]) {
  const V3 d[3] = {normalized(V3{1.0, 0.0137215, 0.0291377}), normalized(V3{0.0173205, 1.0, -0.0262143}),
                   normalized(V3{-0.0119, 0.0233, 1.0})};
  for (int k = 0; k < 3; ++k) {
    dir[k][0] = d[k].x; dir[k][1] = d[k].y; dir[k][2] = d[k].z;
    inv[k][0] = 1.0 / d[k].x; inv[k][1] = 1.0 / d[k].y; inv[k][2] = 1.0 / d[k].z;
  }
}

namespace {
// Eberly's face-integral subexpressions (rigid.cpp:9-21)
void subexpr(double w0, double w1, double w2, double& f1, double& f2, double& f3, double& g0, double& g1,
             double& g2) {
  const double t0 = w0 + w1;
  const double t1 = w0 * w0;
  const double t2 = t1 + w1 * t0;
  f1 = t0 + w2;
  f2 = t2 + w2 * f1;
  f3 = w0 * t1 + w1 * t2 + w2 * f2;
  g0 = f2 + w0 * (f1 + w0);
  g1 = f2 + w1 * (f1 + w1);
  g2 = f2 + w2 * (f1 + w2);
}
}  // namespace

void mesh_inertia(int nv, const double* V, int nf, const int32_t* F, double density, double& mass, double* com,
                  double* I, double* Iinv) {
  if (nv < 4 || nf < 4 || !V || !F) throw std::runtime_error("mesh: needs >= 4 vertices and >= 4 faces");
  const Mesh m{nv, nf, V, F};
  std::vector<double> unused;
  validate(m, unused, false);
  if (density <= 0.0) throw std::invalid_argument("density must be > 0");
  double in[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  const double mult[10] = {1.0 / 6, 1.0 / 24, 1.0 / 24, 1.0 / 24, 1.0 / 60,
                           1.0 / 60, 1.0 / 60, 1.0 / 120, 1.0 / 120, 1.0 / 120};
  for (int f = 0; f < nf; ++f) {
    const V3 p0 = m.v(f, 0), p1 = m.v(f, 1), p2 = m.v(f, 2);
    const V3 d = cross(p1 - p0, p2 - p0);
    double f1x, f2x, f3x, g0x, g1x, g2x, f1y, f2y, f3y, g0y, g1y, g2y, f1z, f2z, f3z, g0z, g1z, g2z;
    subexpr(p0.x, p1.x, p2.x, f1x, f2x, f3x, g0x, g1x, g2x);
    subexpr(p0.y, p1.y, p2.y, f1y, f2y, f3y, g0y, g1y, g2y);
    subexpr(p0.z, p1.z, p2.z, f1z, f2z, f3z, g0z, g1z, g2z);
    in[0] += d.x * f1x;
    in[1] += d.x * f2x;
    in[2] += d.y * f2y;
    in[3] += d.z * f2z;
    in[4] += d.x * f3x;
    in[5] += d.y * f3y;
    in[6] += d.z * f3z;
    in[7] += d.x * (p0.y * g0x + p1.y * g1x + p2.y * g2x);
    in[8] += d.y * (p0.z * g0y + p1.z * g1y + p2.z * g2y);
    in[9] += d.z * (p0.x * g0z + p1.x * g1z + p2.x * g2z);
  }
  for (int i = 0; i < 10; ++i) in[i] *= mult[i];
  const double vol = in[0];
  if (vol <= 0.0) throw std::runtime_error("inertia_from_mesh: non-positive volume");
  mass = density * vol;
  const V3 c = V3{in[1], in[2], in[3]} / vol;
  com[0] = c.x; com[1] = c.y; com[2] = c.z;
  const double xx = in[5] + in[6] - vol * (c.y * c.y + c.z * c.z);
  const double yy = in[4] + in[6] - vol * (c.z * c.z + c.x * c.x);
  const double zz = in[4] + in[5] - vol * (c.x * c.x + c.y * c.y);
  const double xy = -(in[7] - vol * c.x * c.y);
  const double yz = -(in[8] - vol * c.y * c.z);
  const double zx = -(in[9] - vol * c.z * c.x);
  double mI[9] = {xx, xy, zx, xy, yy, yz, zx, yz, zz};
  for (double& e : mI) e *= density;
  for (int k = 0; k < 9; ++k) I[k] = mI[k];
  const double c00 = mI[4] * mI[8] - mI[5] * mI[7];
  const double c01 = mI[5] * mI[6] - mI[3] * mI[8];
  const double c02 = mI[3] * mI[7] - mI[4] * mI[6];
  const double det = mI[0] * c00 + mI[1] * c01 + mI[2] * c02;
  if (!(det > 0.0)) throw std::runtime_error("inertia_from_mesh: inertia tensor not positive definite");
  double inv[9] = {c00, mI[2] * mI[7] - mI[1] * mI[8], mI[1] * mI[5] - mI[2] * mI[4],
                   c01, mI[0] * mI[8] - mI[2] * mI[6], mI[2] * mI[3] - mI[0] * mI[5],
                   c02, mI[1] * mI[6] - mI[0] * mI[7], mI[0] * mI[4] - mI[1] * mI[3]};
  for (int k = 0; k < 9; ++k) Iinv[k] = inv[k] / det;
}

}  // namespace dgx
