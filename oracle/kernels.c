/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into the product path.
 *
 * CPU restatement (plain C, IEEE double, built with -ffp-contract=off) of the
 * three hot-loop contracts of the reference `vmsplat.kernels` module:
 *
 *   oracle_composite_splats   <- pkg/src/vmsplat/kernels/_core.pyx:24-78
 *                                (contract pkg/src/vmsplat/kernels/_ref.py:16-54)
 *   oracle_rasterize_triangles<- pkg/src/vmsplat/kernels/_core.pyx:81-159
 *                                (contract pkg/src/vmsplat/kernels/_ref.py:57-96)
 *   oracle_radix_sort_pairs   <- pkg/src/vmsplat/kernels/_core.pyx:162-202
 *                                (contract pkg/src/vmsplat/kernels/_ref.py:99-112)
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
 * legs may load this library, and only as the checker / the CPU baseline.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_STOP_T (1.0 / 255.0)  /* _core.pyx:20 */
#define ORACLE_MAX_W 0.99            /* _core.pyx:21 */

/* Front-to-back blend of pre-sorted splats into image (h, w, 3) f32, in place.
 * Per pixel: skip once T < 1/255 (test BEFORE blending); weight
 * alpha*exp(sigma) clamped above at 0.99; colour and T stored as f32 after
 * every splat, arithmetic in double (_core.pyx:49-78). */
int oracle_composite_splats(const float *centers, const float *conics,
                            const float *colors, const float *alphas,
                            const int32_t *bounds, int64_t n, float *image,
                            int64_t h, int64_t w) {
  float *trans = (float *)malloc(sizeof(float) * (size_t)(h * w > 0 ? h * w : 1));
  if (!trans) return -1;
  for (int64_t i = 0; i < h * w; ++i) trans[i] = 1.0f;
  for (int64_t i = 0; i < n; ++i) {
    int64_t x0 = bounds[4 * i + 0], x1 = bounds[4 * i + 1];
    int64_t y0 = bounds[4 * i + 2], y1 = bounds[4 * i + 3];
    if (x0 < 0) x0 = 0;
    if (y0 < 0) y0 = 0;
    if (x1 > w) x1 = w;
    if (y1 > h) y1 = h;
    if (x1 <= x0 || y1 <= y0) continue;
    const double cx = centers[2 * i], cy = centers[2 * i + 1];
    const double ca = conics[3 * i], cb = conics[3 * i + 1], cc = conics[3 * i + 2];
    const double al = alphas[i];
    const double cr = colors[3 * i], cg = colors[3 * i + 1], cbl = colors[3 * i + 2];
    for (int64_t y = y0; y < y1; ++y) {
      const double dy = ((double)y + 0.5) - cy;
      for (int64_t x = x0; x < x1; ++x) {
        const int64_t p = y * w + x;
        const double t = trans[p];
        if (t < ORACLE_STOP_T) continue;
        const double dx = ((double)x + 0.5) - cx;
        const double sigma = -0.5 * (ca * dx * dx + 2.0 * cb * dy * dx + cc * dy * dy);
        double wgt = al * exp(sigma);
        if (wgt > ORACLE_MAX_W) wgt = ORACLE_MAX_W;
        float *px = image + 3 * p;
        px[0] = (float)(px[0] + wgt * t * cr);
        px[1] = (float)(px[1] + wgt * t * cg);
        px[2] = (float)(px[2] + wgt * t * cbl);
        trans[p] = (float)(t * (1.0 - wgt));
      }
    }
  }
  free(trans);
  return 0;
}

/* Z-buffered ID raster of screen-space triangles (x, y, 1/z) per corner.
 * Orientation fix (swap b,c when area < 0, skip area == 0), inclusive edge
 * test, strict '>' depth test so the earliest triangle wins exact ties
 * (_core.pyx:105-159).  ids u32, id_image u32 (h, w), invz f64 (h, w). */
int oracle_rasterize_triangles(const double *tris, const uint32_t *ids, int64_t n,
                               uint32_t *id_image, double *invz_image, int64_t h,
                               int64_t w) {
  for (int64_t i = 0; i < n; ++i) {
    const double *t = tris + 9 * i;
    double ax = t[0], ay = t[1], iza = t[2];
    double bx = t[3], by = t[4], izb = t[5];
    double cx = t[6], cy = t[7], izc = t[8];
    double area = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
    if (area == 0.0) continue;
    if (area < 0.0) {
      double s;
      s = bx; bx = cx; cx = s;
      s = by; by = cy; cy = s;
      s = izb; izb = izc; izc = s;
      area = -area;
    }
    double mnx = ax, mxx = ax, mny = ay, mxy = ay;
    if (bx < mnx) mnx = bx;
    if (cx < mnx) mnx = cx;
    if (bx > mxx) mxx = bx;
    if (cx > mxx) mxx = cx;
    if (by < mny) mny = by;
    if (cy < mny) mny = cy;
    if (by > mxy) mxy = by;
    if (cy > mxy) mxy = cy;
    double fx0 = floor(mnx - 0.5), fx1 = ceil(mxx - 0.5);
    double fy0 = floor(mny - 0.5), fy1 = ceil(mxy - 0.5);
    if (fx0 < 0.0) fx0 = 0.0;
    if (fy0 < 0.0) fy0 = 0.0;
    if (fx1 > (double)(w - 1)) fx1 = (double)(w - 1);
    if (fy1 > (double)(h - 1)) fy1 = (double)(h - 1);
    if (fx1 < fx0 || fy1 < fy0) continue;
    const int64_t x0 = (int64_t)fx0, x1 = (int64_t)fx1;
    const int64_t y0 = (int64_t)fy0, y1 = (int64_t)fy1;
    for (int64_t y = y0; y <= y1; ++y) {
      const double py = (double)y + 0.5;
      for (int64_t x = x0; x <= x1; ++x) {
        const double px = (double)x + 0.5;
        const double e0 = (cx - bx) * (py - by) - (cy - by) * (px - bx);
        if (e0 < 0.0) continue;
        const double e1 = (ax - cx) * (py - cy) - (ay - cy) * (px - cx);
        if (e1 < 0.0) continue;
        const double e2 = (bx - ax) * (py - ay) - (by - ay) * (px - ax);
        if (e2 < 0.0) continue;
        const double iz = (e0 * iza + e1 * izb + e2 * izc) / area;
        if (iz > invz_image[y * w + x]) {
          invz_image[y * w + x] = iz;
          id_image[y * w + x] = ids[i];
        }
      }
    }
  }
  return 0;
}

/* Stable ascending LSD radix sort, four 8-bit digits, ping-pong buffers
 * (_core.pyx:162-202).  Sorts keys/values in place. */
int oracle_radix_sort_pairs(uint32_t *keys, int64_t *values, int64_t n) {
  if (n <= 1) return 0;
  uint32_t *k2 = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n);
  int64_t *v2 = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
  if (!k2 || !v2) {
    free(k2);
    free(v2);
    return -1;
  }
  uint32_t *ka = keys, *kb = k2;
  int64_t *va = values, *vb = v2;
  for (int shift = 0; shift < 32; shift += 8) {
    int64_t count[256];
    memset(count, 0, sizeof(count));
    for (int64_t i = 0; i < n; ++i) count[(ka[i] >> shift) & 0xFFu]++;
    int64_t run = 0;
    for (int d = 0; d < 256; ++d) {
      const int64_t c = count[d];
      count[d] = run;
      run += c;
    }
    for (int64_t i = 0; i < n; ++i) {
      const uint32_t d = (ka[i] >> shift) & 0xFFu;
      const int64_t dst = count[d]++;
      kb[dst] = ka[i];
      vb[dst] = va[i];
    }
    uint32_t *kt = ka; ka = kb; kb = kt;
    int64_t *vt = va; va = vb; vb = vt;
  }
  /* four passes: the result is back in the caller's buffers */
  free(k2);
  free(v2);
  return 0;
}

/* Nearest face per point (kernels/_core.pyx:279-334, distance :208-258).
 * Brute force over every face instead of the BVH walk: the reference's
 * answer does not depend on the tree (boxes at equal distance are never
 * pruned, ties go to the lowest face index), so this pins both the distance
 * arithmetic and that claim.  Compiled with -ffp-contract=off like the
 * reference. */
static double o_d2(double x, double y, double z) { return x * x + y * y + z * z; }

static double o_point_tri(double px, double py, double pz, const double *t) {
  double ax = t[0], ay = t[1], az = t[2], bx = t[3], by = t[4], bz = t[5];
  double cx = t[6], cy = t[7], cz = t[8];
  double abx = bx - ax, aby = by - ay, abz = bz - az;
  double acx = cx - ax, acy = cy - ay, acz = cz - az;
  double apx = px - ax, apy = py - ay, apz = pz - az;
  double d1 = abx * apx + aby * apy + abz * apz;
  double d2 = acx * apx + acy * apy + acz * apz;
  if (d1 <= 0.0 && d2 <= 0.0) return o_d2(apx, apy, apz);
  double bpx = px - bx, bpy = py - by, bpz = pz - bz;
  double d3 = abx * bpx + aby * bpy + abz * bpz;
  double d4 = acx * bpx + acy * bpy + acz * bpz;
  if (d3 >= 0.0 && d4 <= d3) return o_d2(bpx, bpy, bpz);
  double vc = d1 * d4 - d3 * d2;
  if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
    double v = d1 / (d1 - d3);
    return o_d2(apx - v * abx, apy - v * aby, apz - v * abz);
  }
  double cpx = px - cx, cpy = py - cy, cpz = pz - cz;
  double d5 = abx * cpx + aby * cpy + abz * cpz;
  double d6 = acx * cpx + acy * cpy + acz * cpz;
  if (d6 >= 0.0 && d5 <= d6) return o_d2(cpx, cpy, cpz);
  double vb = d5 * d2 - d1 * d6;
  if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
    double w = d2 / (d2 - d6);
    return o_d2(apx - w * acx, apy - w * acy, apz - w * acz);
  }
  double va = d3 * d6 - d5 * d4;
  if (va <= 0.0 && (d4 - d3) >= 0.0 && (d5 - d6) >= 0.0) {
    double w = (d4 - d3) / ((d4 - d3) + (d5 - d6));
    return o_d2(px - (bx + w * (cx - bx)), py - (by + w * (cy - by)), pz - (bz + w * (cz - bz)));
  }
  double denom = 1.0 / (va + vb + vc);
  double v = vb * denom, w = vc * denom;
  return o_d2(px - (ax + abx * v + acx * w), py - (ay + aby * v + acy * w),
              pz - (az + abz * v + acz * w));
}

int oracle_nearest_faces(const double *points, int64_t nq, const double *tri_verts,
                         int64_t nf, int64_t *out_face, double *out_dist) {
  for (int64_t q = 0; q < nq; ++q) {
    const double *p = points + 3 * q;
    double best = INFINITY;
    int64_t bf = -1;
    for (int64_t f = 0; f < nf; ++f) {
      double d = o_point_tri(p[0], p[1], p[2], tri_verts + 9 * f);
      if (d < best) { best = d; bf = f; }  /* ascending f: the first minimum wins */
    }
    out_face[q] = bf;
    out_dist[q] = sqrt(best);
  }
  return 0;
}
