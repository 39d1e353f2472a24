/*
 * dgx_mesh.h — triangle-mesh SDF backend (the reference's MeshSdf), FP64,
 * host + device.
 *
 * Same results as the reference's mesh queries on the same mesh, including
 * traversal-order effects:
 *   closest point on a triangle     bvh.cpp:9-60 (Ericson 5.1.5), same op order
 *   BVH                             bvh.cpp:66-103: median split over face
 *                                   centroids on the widest centroid axis, leaf
 *                                   <= 4, DFS preorder node ids. The partition is
 *                                   unique under the (centroid, face id) order, so
 *                                   the host builder (dgx_mesh_host.cu) reproduces
 *                                   the reference's node boxes exactly.
 *   nearest face (within a bound)   bvh.cpp:170-215: near-child DFS, prune on
 *                                   box distance, ties -> lowest face id
 *   sign by ray-crossing parity     bvh.cpp:111-140, 217-254: Moller-Trumbore,
 *                                   slab test, graze -> re-cast along fixed
 *                                   jittered directions
 *   Phong query / dilated_within    sdf.cpp:31-60, 69-81
 * Device code: compiled with --fmad=false, so every product / sum rounds as in
 * the reference's -O3 x86-64 build (no contraction).
 */
#ifndef DGX_MESH_H_
#define DGX_MESH_H_

#include "dgx_geom.h"

namespace dgx {

constexpr int kMeshStack = 48;  // traversal stack; the builder rejects deeper trees (bvh.cpp uses 128)
constexpr int kCertFaces = 24;  // nearest-face certificate: candidate set size cap
constexpr double kCertReach = 5e-3;  // certificate gap search bound (m)
constexpr double kInf = __builtin_huge_val();

#if !defined(DGX_MESH_CNT) || !defined(__CUDA_ARCH__)
#undef DGX_MESH_CNT
#define DGX_MESH_CNT(r, n)
#define DGX_MESH_T(v)
#define DGX_MESH_CYC(r, v)
#else
#define DGX_MESH_T(v) const long long v = clock64()
#define DGX_MESH_CYC(r, v) DGX_MESH_CNT(r, clock64() - (v))
#endif

struct alignas(16) MeshNode {    // 64 B
  double lo[3], hi[3];
  int left, right;   // internal: children; leaf: -1
  int first, count;  // leaf: range of MeshFace records
};

struct alignas(16) MeshFace {    // 80 B, stored in BVH leaf order (bvh.hpp:57 face_order_)
  double a[3], b[3], c[3];  // mesh.v(f, 0..2)
  int f, pad;
};

struct FlatPoint {   // dg::SurfacePoint (bvh.hpp:10-15)
  int face;
  V3 bary, pos;
  double dist2;
};

DGX_GHD double box_dist2(const double* lo, const double* hi, V3 p) {  // Box3::dist2 (vec.hpp:203-211)
  const double v[3] = {p.x, p.y, p.z};
  double d = 0.0;
  for (int i = 0; i < 3; ++i) {
    if (v[i] < lo[i]) { double e = lo[i] - v[i]; d += e * e; }
    else if (v[i] > hi[i]) { double e = v[i] - hi[i]; d += e * e; }
  }
  return d;
}

// bvh.cpp:9-60
DGX_GHD void closest_on_triangle(V3 p, V3 a, V3 b, V3 c, FlatPoint& sp) {
  const V3 ab = b - a, ac = c - a, ap = p - a;
  const double d1 = dot(ab, ap), d2 = dot(ac, ap);
  if (d1 <= 0.0 && d2 <= 0.0) {
    sp.bary = V3{1.0, 0.0, 0.0};
    sp.pos = a;
  } else {
    const V3 bp = p - b;
    const double d3 = dot(ab, bp), d4 = dot(ac, bp);
    if (d3 >= 0.0 && d4 <= d3) {
      sp.bary = V3{0.0, 1.0, 0.0};
      sp.pos = b;
    } else {
      const double vc = d1 * d4 - d3 * d2;
      if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
        const double t = d1 / (d1 - d3);
        sp.bary = V3{1.0 - t, t, 0.0};
        sp.pos = a + t * ab;
      } else {
        const V3 cp = p - c;
        const double d5 = dot(ab, cp), d6 = dot(ac, cp);
        if (d6 >= 0.0 && d5 <= d6) {
          sp.bary = V3{0.0, 0.0, 1.0};
          sp.pos = c;
        } else {
          const double vb = d5 * d2 - d1 * d6;
          if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
            const double t = d2 / (d2 - d6);
            sp.bary = V3{1.0 - t, 0.0, t};
            sp.pos = a + t * ac;
          } else {
            const double va = d3 * d6 - d5 * d4;
            if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
              const double t = (d4 - d3) / ((d4 - d3) + (d5 - d6));
              sp.bary = V3{0.0, 1.0 - t, t};
              sp.pos = b + t * (c - b);
            } else {
              const double denom = 1.0 / (va + vb + vc);
              const double v = vb * denom, w = vc * denom;
              sp.bary = V3{1.0 - v - w, v, w};
              sp.pos = a + v * ab + w * ac;
            }
          }
        }
      }
    }
  }
  sp.dist2 = dot(p - sp.pos, p - sp.pos);
}

// read-only loads through the non-coherent path on the device
DGX_GHD MeshNode load_node(const MeshNode* p) {
#if defined(__CUDA_ARCH__)
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  const int4 d = __ldg(reinterpret_cast<const int4*>(p) + 3);
  MeshNode n;
  n.lo[0] = a.x; n.lo[1] = a.y; n.lo[2] = b.x;
  n.hi[0] = b.y; n.hi[1] = c.x; n.hi[2] = c.y;
  n.left = d.x; n.right = d.y; n.first = d.z; n.count = d.w;
  return n;
#else
  return *p;
#endif
}

DGX_GHD double node_lb2(const MeshNode* p, V3 r) {
#if defined(__CUDA_ARCH__)
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  const double lo[3] = {a.x, a.y, b.x}, hi[3] = {b.y, c.x, c.y};
  return box_dist2(lo, hi, r);
#else
  return box_dist2(p->lo, p->hi, r);
#endif
}

DGX_GHD void node_links(const MeshNode* p, int& left, int& right, int& first, int& count) {
#if defined(__CUDA_ARCH__)
  const int4 d = __ldg(reinterpret_cast<const int4*>(p) + 3);
  left = d.x; right = d.y; first = d.z; count = d.w;
#else
  left = p->left; right = p->right; first = p->first; count = p->count;
#endif
}

struct FaceV {
  V3 a, b, c;
  int f;
};

DGX_GHD FaceV load_face(const MeshFace* p) {
#if defined(__CUDA_ARCH__)
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 x0 = __ldg(q), x1 = __ldg(q + 1), x2 = __ldg(q + 2), x3 = __ldg(q + 3);
  const double c2 = __ldg(reinterpret_cast<const double*>(p) + 8);
  const int f = __ldg(&p->f);
  return FaceV{V3{x0.x, x0.y, x1.x}, V3{x1.y, x2.x, x2.y}, V3{x3.x, x3.y, c2}, f};
#else
  return FaceV{V3{p->a[0], p->a[1], p->a[2]}, V3{p->b[0], p->b[1], p->b[2]}, V3{p->c[0], p->c[1], p->c[2]}, p->f};
#endif
}

DGX_GHD V3 load_v3(const double* p) {
#if defined(__CUDA_ARCH__)
  return V3{__ldg(p), __ldg(p + 1), __ldg(p + 2)};
#else
  return V3{p[0], p[1], p[2]};
#endif
}

DGX_GHD int load_i(const int* p) {
#if defined(__CUDA_ARCH__)
  return __ldg(p);
#else
  return *p;
#endif
}

// Mesh geometry + constants; resident in device global memory (one copy per
// uploaded object), reached through MeshSdf::g.
struct MeshGeom {
  const MeshNode* nodes;
  const MeshFace* faces;
  const int* tri;        // [F,3] vertex ids (mesh.faces)
  const double* vn;      // [V,3] vertex normals (mesh.vertex_normals)
  const double* vx;      // [V,3] vertices
  double blo[3], bhi[3]; // mesh bounds (TriMesh::bounds, all vertices)
  double alpha;          // alpha_phong
  double dir[3][3];      // ray directions kRayDir0, kRayDir1, third fixed direction (bvh.cpp:143-144, 250)
  double inv[3][3];      // 1 / dir, per component (bvh.cpp:219)
  double cull;           // ContactSolver::kCullMargin (sim.hpp:213)
  const int* vf_off;     // [V+1] vertex -> incident faces (CSR), for certificates
  const int* vf_idx;
  int nfaces;

  DGX_GHD MeshNode node(int i) const { return load_node(nodes + i); }

  // closest point on face f (mesh.v(f, 0..2), bvh.cpp:193)
  DGX_GHD void face_closest(V3 r, int f, FlatPoint& sp) const {
    const int i0 = load_i(tri + 3 * f), i1 = load_i(tri + 3 * f + 1), i2 = load_i(tri + 3 * f + 2);
    closest_on_triangle(r, load_v3(vx + 3 * i0), load_v3(vx + 3 * i1), load_v3(vx + 3 * i2), sp);
    sp.face = f;
  }

  // Solver-path nearest face: the same argmin (dist2, then lowest face id) as
  // nearest(), seeded with a hint face (the point's face one sweep earlier;
  // any id, or -1) so the first prune bound is already tight. Pruning keeps a
  // relative + absolute slack over the rounded triangle distances, so no box
  // holding the argmin is skipped; the result is the exact argmin over all
  // faces (what the reference's traversal returns barring its own rounding
  // ties at a box boundary).
  DGX_GHD void nearest_ws(V3 r, int hint, FlatPoint& best) const {
    double best2 = kInf;
    best.face = -1;
    if (hint >= 0 && hint < nfaces) {
      face_closest(r, hint, best);
      best2 = best.dist2;
    }
    // stack of (node, its lower bound computed when its parent was expanded)
    int stack[kMeshStack];
    double sb[kMeshStack];
    int top = 0;
    stack[top] = 0;
    sb[top++] = node_lb2(nodes, r);
    DGX_MESH_CNT(23, 1);
    while (top > 0) {
      --top;
      const double lim = best2 * (1.0 + 1e-10) + 1e-24;
      if (sb[top] > lim) continue;
      const int id = stack[top];
      DGX_MESH_CNT(24, 1);
      int left, right, first, count;
      node_links(nodes + id, left, right, first, count);
      if (left < 0) {
        for (int i = first; i < first + count; ++i) {
          const FaceV F = load_face(faces + i);
          FlatPoint sp;
          closest_on_triangle(r, F.a, F.b, F.c, sp);
          if (sp.dist2 < best2 || (sp.dist2 == best2 && (best.face < 0 || F.f < best.face))) {
            best2 = sp.dist2;
            best = sp;
            best.face = F.f;
          }
        }
      } else {
        const double dl = node_lb2(nodes + left, r), dr = node_lb2(nodes + right, r);
        if (dl <= dr) {  // nearer child on top
          if (dr <= lim) { stack[top] = right; sb[top++] = dr; }
          if (dl <= lim) { stack[top] = left; sb[top++] = dl; }
        } else {
          if (dl <= lim) { stack[top] = left; sb[top++] = dl; }
          if (dr <= lim) { stack[top] = right; sb[top++] = dr; }
        }
      }
    }
  }

  // Bvh::closest_point_within (bvh.cpp:170-215); limit2 = max_dist^2 or +inf.
  // Returns false when no face is within the bound. Same traversal order and
  // box pruning as the reference.
  DGX_GHD bool nearest(V3 r, double limit2, FlatPoint& best) const {
    double best2 = limit2;
    best.face = -1;
    int stack[kMeshStack];
    int top = 0;
    const MeshNode root = node(0);
    if (box_dist2(root.lo, root.hi, r) > best2) return false;
    stack[top++] = 0;
    DGX_MESH_CNT(23, 1);
    while (top > 0) {
      const int id = stack[--top];
      const MeshNode nd = node(id);
      DGX_MESH_CNT(24, 1);
      if (box_dist2(nd.lo, nd.hi, r) > best2) continue;  // e.d2 > best2 (same value as at push time)
      if (nd.left < 0) {
        for (int i = nd.first; i < nd.first + nd.count; ++i) {
          const FaceV F = load_face(faces + i);
          FlatPoint sp;
          closest_on_triangle(r, F.a, F.b, F.c, sp);
          sp.face = F.f;
          if (sp.dist2 < best2 || (sp.dist2 == best2 && (best.face < 0 || F.f < best.face))) {
            best2 = sp.dist2;
            best = sp;
          }
        }
      } else {
        const MeshNode L = node(nd.left), R = node(nd.right);
        const double dl = box_dist2(L.lo, L.hi, r), dr = box_dist2(R.lo, R.hi, r);
        if (dl <= dr) {
          if (dr <= best2) stack[top++] = nd.right;
          if (dl <= best2) stack[top++] = nd.left;
        } else {
          if (dl <= best2) stack[top++] = nd.left;
          if (dr <= best2) stack[top++] = nd.right;
        }
      }
    }
    return best.face >= 0;
  }

  // ray_box (bvh.cpp:129-140), std::max / std::min semantics
  DGX_GHD static bool ray_box(V3 o, const double* inv, const double* lo, const double* hi) {
    const double ov[3] = {o.x, o.y, o.z};
    double t0 = 0.0, t1 = kInf;
    for (int i = 0; i < 3; ++i) {
      double ta = (lo[i] - ov[i]) * inv[i];
      double tb = (hi[i] - ov[i]) * inv[i];
      if (ta > tb) { double s = ta; ta = tb; tb = s; }
      t0 = (t0 < ta) ? ta : t0;
      t1 = (tb < t1) ? tb : t1;
      if (t0 > t1) return false;
    }
    return true;
  }

  // Bvh::count_ray_crossings (bvh.cpp:217-241): -1 = a hit grazed a feature
  DGX_GHD int count_crossings(V3 o, int k) const {
    const V3 d{dir[k][0], dir[k][1], dir[k][2]};
    int count = 0;
    int stack[kMeshStack];
    int top = 0;
    stack[top++] = 0;
    DGX_MESH_CNT(25, 1);
    while (top > 0) {
      const MeshNode nd = node(stack[--top]);
      DGX_MESH_CNT(26, 1);
      if (!ray_box(o, inv[k], nd.lo, nd.hi)) continue;
      if (nd.left < 0) {
        for (int i = nd.first; i < nd.first + nd.count; ++i) {
          const FaceV F = load_face(faces + i);
          // ray_triangle (bvh.cpp:111-127)
          const V3 a = F.a;
          const V3 e1 = F.b - a, e2 = F.c - a;
          const V3 h = cross(d, e2);
          const double det = dot(e1, h);
          if ((det < 0.0 ? -det : det) < 1e-14) continue;
          const double f = 1.0 / det;
          const V3 s = o - a;
          const double u = f * dot(s, h);
          const V3 q = cross(s, e1);
          const double v = f * dot(d, q);
          const double w = 1.0 - u - v;
          if (u < 0.0 || v < 0.0 || w < 0.0) continue;
          const double t = f * dot(e2, q);
          if (t <= 0.0) continue;
          double mb = u;
          if (v < mb) mb = v;
          if (w < mb) mb = w;
          if (mb < 1e-12 || t < 1e-12) return -1;  // feature graze
          ++count;
        }
      } else {
        stack[top++] = nd.left;
        stack[top++] = nd.right;
      }
    }
    return count;
  }

  // Bvh::sign_at (bvh.cpp:243-254)
  DGX_GHD int sign_at(V3 r) const {
    int c = count_crossings(r, 0);
    if (c < 0) c = count_crossings(r, 1);
    if (c < 0) c = count_crossings(r, 2);
    if (c < 0) return 1;
    return (c % 2 == 0) ? 1 : -1;
  }

  DGX_GHD SdfQuery phong(V3 r, const FlatPoint& fl) const {
    return phong_signed(r, fl, dsqrt(fl.dist2) < kSurfaceEps ? 1 : sign_at(r));
  }

  // MeshSdf::phong(r, alpha_) (sdf.cpp:31-60) from a flat closest point and
  // the sign of sdf.cpp:47
  DGX_GHD SdfQuery phong_signed(V3 r, const FlatPoint& fl, int sign) const {
    const int t[3] = {load_i(tri + 3 * fl.face), load_i(tri + 3 * fl.face + 1), load_i(tri + 3 * fl.face + 2)};
    const V3 rstar = fl.pos;
    SdfQuery q;
    if (alpha == 0.0) {
      q.proxy = rstar;
    } else {
      V3 pp[3];
      for (int k = 0; k < 3; ++k) {  // plane_project (sdf.cpp:12-14)
        const V3 v = load_v3(vx + 3 * t[k]), n = load_v3(vn + 3 * t[k]);
        pp[k] = rstar - dot(rstar - v, n) * n;
      }
      const V3 blend = fl.bary.x * pp[0] + fl.bary.y * pp[1] + fl.bary.z * pp[2];
      q.proxy = (1.0 - alpha) * rstar + alpha * blend;
    }
    q.sign = sign;
    const V3 delta = r - q.proxy;
    const double d = norm(delta);
    q.rho = static_cast<double>(q.sign) * d;
    if (d < kSurfaceEps) {
      const V3 n = fl.bary.x * load_v3(vn + 3 * t[0]) + fl.bary.y * load_v3(vn + 3 * t[1]) + fl.bary.z * load_v3(vn + 3 * t[2]);
      q.grad = normalized(n);
    } else {
      q.grad = (static_cast<double>(q.sign) / d) * delta;
    }
    return q;
  }

  DGX_GHD SdfQuery query(V3 r) const {
    DGX_MESH_CNT(27, 1);
    FlatPoint fl;
    nearest(r, kInf, fl);
    return phong(r, fl);
  }

  // Faces incident to any vertex of face f, sorted; -1 if more than cap.
  DGX_GHD int ring_faces(int f, int* out, int cap) const {
    int n = 0;
    for (int k = 0; k < 3; ++k) {
      const int v = load_i(tri + 3 * f + k);
      const int b = load_i(vf_off + v), e = load_i(vf_off + v + 1);
      for (int j = b; j < e; ++j) {
        const int g = load_i(vf_idx + j);
        bool seen = false;
        for (int t = 0; t < n; ++t) seen = seen || out[t] == g;
        if (seen) continue;
        if (n == cap) return -1;
        int t = n++;
        while (t > 0 && out[t - 1] > g) { out[t] = out[t - 1]; --t; }
        out[t] = g;
      }
    }
    return n;
  }

  // Smallest squared distance from r over faces NOT in the sorted set C (n),
  // or lim2 when none is closer (box-pruned traversal)
  DGX_GHD double nearest_excluding(V3 r, const int* C, int n, double lim2) const {
    double best2 = lim2;
    int stack[kMeshStack];
    double sb[kMeshStack];
    int top = 0;
    stack[top] = 0;
    sb[top++] = node_lb2(nodes, r);
    while (top > 0) {
      --top;
      if (sb[top] > best2) continue;
      int left, right, first, count;
      node_links(nodes + stack[top], left, right, first, count);
      if (left < 0) {
        for (int i = first; i < first + count; ++i) {
          const FaceV F = load_face(faces + i);
          int lo = 0, hi = n;  // binary search in C
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (C[mid] < F.f) lo = mid + 1; else hi = mid;
          }
          if (lo < n && C[lo] == F.f) continue;
          FlatPoint sp;
          closest_on_triangle(r, F.a, F.b, F.c, sp);
          if (sp.dist2 < best2) best2 = sp.dist2;
        }
      } else {
        const double dl = node_lb2(nodes + left, r), dr = node_lb2(nodes + right, r);
        if (dl <= dr) {
          if (dr <= best2) { stack[top] = right; sb[top++] = dr; }
          if (dl <= best2) { stack[top] = left; sb[top++] = dl; }
        } else {
          if (dl <= best2) { stack[top] = left; sb[top++] = dl; }
          if (dr <= best2) { stack[top] = right; sb[top++] = dr; }
        }
      }
    }
    return best2;
  }

  // Solver forward with a per-point nearest-face certificate (cert: rc.x,
  // rc.y, rc.z, rad; cf: n then n sorted face ids). Valid while |r - rc| <
  // rad: every face outside the set is then strictly farther than the
  // certified nearest face, so the argmin (dist2, lowest id) over the set IS
  // the global one. Otherwise the point is re-certified: warm-started nearest
  // search, the set = faces around the nearest face's vertices, g = nearest
  // distance outside the set (searched up to d + kCertReach), rad = (g - d)/2
  // less a rounding allowance. The sign always comes from the ray cast.
  DGX_GHD SdfQuery query_cert(V3 r, int hint, int& packed, double* cert, int* cf) const {
    FlatPoint fl;
    fl.face = -1;
    const double rad = cert[3];
    DGX_MESH_T(tq0);
    if (rad > 0.0) {
      const V3 dv = V3{r.x - cert[0], r.y - cert[1], r.z - cert[2]};
      if (dot(dv, dv) < rad * rad) {
        DGX_MESH_CNT(28, 1);
        const int n = cf[0];
        double best2 = kInf;
        for (int t = 0; t < n; ++t) {
          const int f = cf[1 + t];  // ascending ids: a tie keeps the lower id
          FlatPoint sp;
          face_closest(r, f, sp);
          if (sp.dist2 < best2) {
            best2 = sp.dist2;
            fl = sp;
          }
        }
      }
    }
    DGX_MESH_CYC(29, tq0);
    DGX_MESH_T(tq1);
    if (fl.face < 0) {
      nearest_ws(r, hint, fl);
      int C[kCertFaces];
      const int n = ring_faces(fl.face, C, kCertFaces);
      cert[3] = -1.0;
      if (n > 0) {
        const double d = dsqrt(fl.dist2);
        const double lim = d + kCertReach;
        const double g = dsqrt(nearest_excluding(r, C, n, lim * lim));
        const double rr = 0.5 * (g - d) - (1e-12 + 1e-9 * (g + d));
        if (rr > 0.0) {
          cert[0] = r.x; cert[1] = r.y; cert[2] = r.z; cert[3] = rr;
          cf[0] = n;
          for (int t = 0; t < n; ++t) cf[1 + t] = C[t];
        }
      }
    }
    DGX_MESH_CYC(30, tq1);
    DGX_MESH_T(tq2);
    const SdfQuery q = phong(r, fl);
    DGX_MESH_CYC(31, tq2);
    packed = (fl.face << 1) | (q.sign < 0 ? 1 : 0);
    return q;
  }

  // solver forward: query via nearest_ws; *packed = face << 1 | (sign < 0)
  DGX_GHD SdfQuery query_ws(V3 r, int hint, int& packed) const {
    DGX_MESH_CNT(27, 1);
    FlatPoint fl;
    nearest_ws(r, hint, fl);
    const SdfQuery q = phong(r, fl);
    packed = (fl.face << 1) | (q.sign < 0 ? 1 : 0);
    return q;
  }

  // solver adjoint: the forward's query at the same r re-evaluated from its
  // packed (face, sign) — one triangle instead of a traversal + ray cast
  DGX_GHD SdfQuery query_packed(V3 r, int packed) const {
    FlatPoint fl;
    face_closest(r, packed >> 1, fl);
    return phong_signed(r, fl, (packed & 1) ? -1 : 1);
  }

  // dilated_within's cull (sdf.cpp:69-77): true = nullopt (sample culled)
  DGX_GHD bool culled(V3 r, double radius) const {
    const double md = radius + cull;
    FlatPoint fl;
    if (nearest(r, md * md, fl)) return false;
    return box_dist2(blo, bhi, r) > 0.0 || sign_at(r) > 0;
  }
};

// Kernel-facing handle (8 B kernel parameter). The traversal is kept out of
// line so the fused kernel's register allocation is not driven by it.
struct MeshSdf {
  const MeshGeom* g;
#if defined(__CUDACC__)
  __device__ SdfQuery query(V3 r) const;
  __device__ bool culled(V3 r, double radius) const;
  __device__ SdfQuery query_ws(V3 r, int hint, int& packed) const;
  __device__ SdfQuery query_packed(V3 r, int packed) const;
  __device__ SdfQuery query_cert(V3 r, int hint, int& packed, double* cert, int* cf) const;
#endif
};

#if defined(__CUDACC__)
static __device__ __noinline__ SdfQuery mesh_query(const MeshGeom* __restrict__ g, V3 r) { return g->query(r); }
static __device__ __noinline__ bool mesh_culled(const MeshGeom* __restrict__ g, V3 r, double radius) {
  return g->culled(r, radius);
}
static __device__ __noinline__ SdfQuery mesh_query_ws(const MeshGeom* __restrict__ g, V3 r, int hint, int* packed) {
  return g->query_ws(r, hint, *packed);
}
static __device__ __noinline__ SdfQuery mesh_query_packed(const MeshGeom* __restrict__ g, V3 r, int packed) {
  return g->query_packed(r, packed);
}
static __device__ __noinline__ SdfQuery mesh_query_cert(const MeshGeom* __restrict__ g, V3 r, int hint, int* packed,
                                                       double* cert, int* cf) {
  return g->query_cert(r, hint, *packed, cert, cf);
}
__device__ __forceinline__ SdfQuery MeshSdf::query_cert(V3 r, int hint, int& packed, double* cert, int* cf) const {
  return mesh_query_cert(g, r, hint, &packed, cert, cf);
}
__device__ __forceinline__ SdfQuery MeshSdf::query(V3 r) const { return mesh_query(g, r); }
__device__ __forceinline__ SdfQuery MeshSdf::query_ws(V3 r, int hint, int& packed) const {
  return mesh_query_ws(g, r, hint, &packed);
}
__device__ __forceinline__ SdfQuery MeshSdf::query_packed(V3 r, int packed) const {
  return mesh_query_packed(g, r, packed);
}
__device__ __forceinline__ bool MeshSdf::culled(V3 r, double radius) const { return mesh_culled(g, r, radius); }
#endif

}  // namespace dgx

#endif  // DGX_MESH_H_
