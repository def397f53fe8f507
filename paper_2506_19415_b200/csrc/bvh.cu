// SURVEY §8(f) F3, preprocessing accelerator: nearest proxy-mesh face per
// query point over a flat median-split BVH - the reference's
// bvh_nearest_points (pkg/src/vmsplat/kernels/_core.pyx:279-334), used by the
// page builder's link sampling (pkg/src/vmsplat/paging.py:336) and record
// assignment (paging.py:68).
//
// One thread per query point; the traversal (depth-first, nearer child
// popped first, subtrees pruned when their box is strictly farther than the
// best face so far) and the distance arithmetic are the reference's, in FP64
// with every product and sum rounded separately (the reference is compiled
// with -ffp-contract=off, pkg/setup.py:22) - so faces and distances are
// bit-identical.  Ties resolve to the lowest face index; because equal-
// distance boxes are never pruned, the answer does not depend on the tree.
#include "common.cuh"

namespace vms {
namespace {

constexpr int kBvhStack = 128;  // the reference's fixed traversal stack

VMS_DEV double dist2(double x, double y, double z) {
  return dadd(dadd(dmul(x, x), dmul(y, y)), dmul(z, z));
}

VMS_DEV double dot3n(double ax, double ay, double az, double bx, double by, double bz) {
  return dadd(dadd(dmul(ax, bx), dmul(ay, by)), dmul(az, bz));
}

// Ericson's closest point on a triangle, squared distance (_core.pyx:208-258).
__device__ double point_tri_dist2(double px, double py, double pz,
                                  const double* __restrict__ t) {
  const double ax = t[0], ay = t[1], az = t[2];
  const double bx = t[3], by = t[4], bz = t[5];
  const double cx = t[6], cy = t[7], cz = t[8];
  const double abx = dsub(bx, ax), aby = dsub(by, ay), abz = dsub(bz, az);
  const double acx = dsub(cx, ax), acy = dsub(cy, ay), acz = dsub(cz, az);
  const double apx = dsub(px, ax), apy = dsub(py, ay), apz = dsub(pz, az);
  const double d1 = dot3n(abx, aby, abz, apx, apy, apz);
  const double d2 = dot3n(acx, acy, acz, apx, apy, apz);
  if (d1 <= 0.0 && d2 <= 0.0) return dist2(apx, apy, apz);  // vertex a
  const double bpx = dsub(px, bx), bpy = dsub(py, by), bpz = dsub(pz, bz);
  const double d3 = dot3n(abx, aby, abz, bpx, bpy, bpz);
  const double d4 = dot3n(acx, acy, acz, bpx, bpy, bpz);
  if (d3 >= 0.0 && d4 <= d3) return dist2(bpx, bpy, bpz);  // vertex b
  const double vc = dsub(dmul(d1, d4), dmul(d3, d2));
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {  // edge ab
    const double v = ddiv(d1, dsub(d1, d3));
    return dist2(dsub(apx, dmul(v, abx)), dsub(apy, dmul(v, aby)), dsub(apz, dmul(v, abz)));
  }
  const double cpx = dsub(px, cx), cpy = dsub(py, cy), cpz = dsub(pz, cz);
  const double d5 = dot3n(abx, aby, abz, cpx, cpy, cpz);
  const double d6 = dot3n(acx, acy, acz, cpx, cpy, cpz);
  if (d6 >= 0.0 && d5 <= d6) return dist2(cpx, cpy, cpz);  // vertex c
  const double vb = dsub(dmul(d5, d2), dmul(d1, d6));
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {  // edge ac
    const double w = ddiv(d2, dsub(d2, d6));
    return dist2(dsub(apx, dmul(w, acx)), dsub(apy, dmul(w, acy)), dsub(apz, dmul(w, acz)));
  }
  const double va = dsub(dmul(d3, d6), dmul(d5, d4));
  const double e43 = dsub(d4, d3), e56 = dsub(d5, d6);
  if (va <= 0.0 && e43 >= 0.0 && e56 >= 0.0) {  // edge bc
    const double w = ddiv(e43, dadd(e43, e56));
    const double qx = dadd(bx, dmul(w, dsub(cx, bx)));
    const double qy = dadd(by, dmul(w, dsub(cy, by)));
    const double qz = dadd(bz, dmul(w, dsub(cz, bz)));
    return dist2(dsub(px, qx), dsub(py, qy), dsub(pz, qz));
  }
  const double denom = ddiv(1.0, dadd(dadd(va, vb), vc));  // interior
  const double v = dmul(vb, denom), w = dmul(vc, denom);
  const double qx = dadd(dadd(ax, dmul(abx, v)), dmul(acx, w));
  const double qy = dadd(dadd(ay, dmul(aby, v)), dmul(acy, w));
  const double qz = dadd(dadd(az, dmul(abz, v)), dmul(acz, w));
  return dist2(dsub(px, qx), dsub(py, qy), dsub(pz, qz));
}

// Squared distance from the point to a node's box (0 inside; _core.pyx:261-276).
VMS_DEV double aabb_dist2(double px, double py, double pz, const double* __restrict__ b) {
  double acc = 0.0, d;
  d = dsub(b[0], px);
  if (d < 0.0) d = dsub(px, b[3]);
  if (d > 0.0) acc = dadd(acc, dmul(d, d));
  d = dsub(b[1], py);
  if (d < 0.0) d = dsub(py, b[4]);
  if (d > 0.0) acc = dadd(acc, dmul(d, d));
  d = dsub(b[2], pz);
  if (d < 0.0) d = dsub(pz, b[5]);
  if (d > 0.0) acc = dadd(acc, dmul(d, d));
  return acc;
}

__global__ void __launch_bounds__(128) bvh_nearest_k(
    const double* __restrict__ points, int64_t nq, const double* __restrict__ bounds,
    const int2* __restrict__ children, const int2* __restrict__ ranges,
    const int32_t* __restrict__ tri_order, const double* __restrict__ tri_verts,
    int64_t* __restrict__ out_face, double* __restrict__ out_dist, int32_t* overflow) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const double px = points[3 * q], py = points[3 * q + 1], pz = points[3 * q + 2];
  double best = __longlong_as_double(0x7ff0000000000000ll);  // +inf
  int64_t best_face = -1;
  int stack[kBvhStack];
  int sp = 0;
  stack[sp++] = 0;
  while (sp > 0) {
    const int node = stack[--sp];
    if (aabb_dist2(px, py, pz, bounds + 6 * (size_t)node) > best) continue;
    const int2 ch = children[node];
    if (ch.x < 0) {
      const int2 r = ranges[node];
      for (int k = r.x; k < r.y; ++k) {
        const int64_t face = tri_order[k];
        const double d2 = point_tri_dist2(px, py, pz, tri_verts + 9 * (size_t)face);
        if (d2 < best || (d2 == best && face < best_face)) {
          best = d2;
          best_face = face;
        }
      }
    } else {
      if (sp + 2 > kBvhStack) {
        atomicExch(overflow, 1);
        best_face = -1;
        break;
      }
      const double dl = aabb_dist2(px, py, pz, bounds + 6 * (size_t)ch.x);
      const double dr = aabb_dist2(px, py, pz, bounds + 6 * (size_t)ch.y);
      // the farther child goes first, so the nearer one pops first
      stack[sp] = dl <= dr ? ch.y : ch.x;
      stack[sp + 1] = dl <= dr ? ch.x : ch.y;
      sp += 2;
    }
  }
  out_face[q] = best_face;
  out_dist[q] = __dsqrt_rn(best);
}

}  // namespace
}  // namespace vms

extern "C" int32_t vms_bvh_nearest_points(const double* points, int64_t n_points,
                                          const double* bounds, const int32_t* children,
                                          const int32_t* ranges, int64_t n_nodes,
                                          const int32_t* tri_order, const double* tri_verts,
                                          int64_t n_faces, int64_t* out_face, double* out_dist,
                                          int32_t* overflow, void* stream) {
  using namespace vms;
  if (n_points < 0 || n_nodes < 1 || n_faces < 1 || !bounds || !children || !ranges ||
      !tri_order || !tri_verts || !overflow ||
      (n_points > 0 && (!points || !out_face || !out_dist))) {
    set_error("bvh_nearest_points: invalid arguments");
    return VMS_ERR_INVALID;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  VMS_CUDA(cudaMemsetAsync(overflow, 0, sizeof(int32_t), s));
  if (n_points == 0) return VMS_OK;
  const int T = 128;
  bvh_nearest_k<<<(unsigned)ceil_div<int64_t>(n_points, T), T, 0, s>>>(
      points, n_points, bounds, reinterpret_cast<const int2*>(children),
      reinterpret_cast<const int2*>(ranges), tri_order, tri_verts, out_face, out_dist, overflow);
  mark("bvh_nearest", s);
  VMS_LAUNCH_CHECK("bvh_nearest_points");
  return VMS_OK;
}
