// Subsystem [4]: 3DGS preprocessing over the resident pages only.
// Compiled with -fmad=false; FP64 throughout, NumPy elementwise semantics
// (one rounding per operation) and the probed BLAS dot order for every
// matrix product, following pkg/src/vmsplat/render.py:104-220 and the cull
// of compute_keys (render.py:138-152).
//
// One CTA per resident-page chunk (<= 128 records, 30 KB).  The chunk's AoS
// rows (59 f32 = 236 B each) are staged into shared memory with coalesced
// 16-byte loads; record stride 59 words is odd, so the per-thread column
// reads that follow are bank-conflict free.
#include <algorithm>

#include "common.cuh"
#include "render.h"

namespace vms {

namespace {

// render.py:23-44
constexpr double kLowPass = 0.3;
constexpr double kMinDet = 1e-12;
constexpr double kExtentSigma = 3.0;
constexpr double C0 = 0.28209479177387814;
constexpr double C1 = 0.4886025119029199;
constexpr double C2_0 = 1.0925484305920792, C2_1 = -1.0925484305920792,
                 C2_2 = 0.31539156525252005, C2_3 = -1.0925484305920792,
                 C2_4 = 0.5462742152960396;
constexpr double C3_0 = -0.5900435899266435, C3_1 = 2.890611442640554,
                 C3_2 = -0.4570457994644658, C3_3 = 0.3731763325901154,
                 C3_4 = -0.4570457994644658, C3_5 = 1.445305721320277,
                 C3_6 = -0.5900435899266435;

// gaussians.quat_to_matrix, (w, x, y, z) -> row-major R (gaussians.py:76-96)
__device__ __forceinline__ void quat_rot(double w, double x, double y, double z, double* m) {
  m[0] = 1.0 - 2.0 * (y * y + z * z);
  m[1] = 2.0 * (x * y - w * z);
  m[2] = 2.0 * (x * z + w * y);
  m[3] = 2.0 * (x * y + w * z);
  m[4] = 1.0 - 2.0 * (x * x + z * z);
  m[5] = 2.0 * (y * z - w * x);
  m[6] = 2.0 * (x * z - w * y);
  m[7] = 2.0 * (y * z + w * x);
  m[8] = 1.0 - 2.0 * (x * x + y * y);
}

// Degree-3 SH -> RGB for one unit direction (render.py:104-135); coef is
// coefficient-major (c * 3 + ch), stride `cs` between coefficients.
template <typename CoefT>
__device__ __forceinline__ void sh_rgb(const CoefT* coef, double vx, double vy, double vz,
                                       double* col) {
  const double xx = vx * vx, yy = vy * vy, zz = vz * vz;
  const double xy = vx * vy, yz = vy * vz, xz = vx * vz;
  double basis[16];
  basis[0] = C0;
  basis[1] = (-C1) * vy;
  basis[2] = C1 * vz;
  basis[3] = (-C1) * vx;
  basis[4] = C2_0 * xy;
  basis[5] = C2_1 * yz;
  basis[6] = C2_2 * ((2.0 * zz - xx) - yy);
  basis[7] = C2_3 * xz;
  basis[8] = C2_4 * (xx - yy);
  basis[9] = (C3_0 * vy) * (3.0 * xx - yy);
  basis[10] = (C3_1 * xy) * vz;
  basis[11] = (C3_2 * vy) * ((4.0 * zz - xx) - yy);
  basis[12] = (C3_3 * vz) * ((2.0 * zz - 3.0 * xx) - 3.0 * yy);
  basis[13] = (C3_4 * vx) * ((4.0 * zz - xx) - yy);
  basis[14] = (C3_5 * vz) * (xx - yy);
  basis[15] = (C3_6 * vx) * (xx - 3.0 * yy);
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) {
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) acc = acc + basis[k] * (double)coef[3 * k + ch];
    col[ch] = fmax(0.5 + acc, 0.0);
  }
}

struct Proj {
  double tz;           // view depth (key source)
  double cx, cy;       // pixel centre
  double ca, cb, cc;   // conic (c/det, -b/det, a/det)
  double col[3];
  int x0, x1, y0, y1;  // half-open pixel bounds
  bool live;           // compute_keys cull passed
  bool kept;           // project_records cull passed
};

// compute_keys cull + project_records for one record r[59] (render.py:138-220).
__device__ __forceinline__ void project_one(const float* r, const RenderCamera& cam, Proj& o,
                                            bool cull_live) {
  const double d0 = (double)r[0] - cam.pos[0], d1 = (double)r[1] - cam.pos[1],
               d2 = (double)r[2] - cam.pos[2];
  const int dm = cam.dot_mode;
  const double tx = dot3(dm, d0, d1, d2, cam.rot[0], cam.rot[3], cam.rot[6]);
  const double ty = dot3(dm, d0, d1, d2, cam.rot[1], cam.rot[4], cam.rot[7]);
  const double tz = dot3(dm, d0, d1, d2, cam.rot[2], cam.rot[5], cam.rot[8]);
  o.tz = tz;
  o.live = r[10] > 0.0f && tz > cam.near;
  o.kept = false;
  if (cull_live && !o.live) return;
  double R[9];
  quat_rot((double)r[3], (double)r[4], (double)r[5], (double)r[6], R);
  const double sx = r[7], sy = r[8], sz = r[9];
  double ms[9];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    ms[3 * i + 0] = R[3 * i + 0] * sx;
    ms[3 * i + 1] = R[3 * i + 1] * sy;
    ms[3 * i + 2] = R[3 * i + 2] * sz;
  }
  double cov3[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      cov3[3 * i + k] =
          dot3(dm, ms[3 * i], ms[3 * i + 1], ms[3 * i + 2], ms[3 * k], ms[3 * k + 1], ms[3 * k + 2]);
  const double f = cam.focal;
  const double tz2 = tz * tz;
  const double j00 = f / tz, j02 = (-f * tx) / tz2;
  const double j11 = f / tz, j12 = (-f * ty) / tz2;
  // jw = J @ cam_rot.T : jw[r][c] = sum_k J[r][k] * rot[c][k]
  double jw[6];
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    jw[c] = dot3(dm, j00, 0.0, j02, cam.rot[3 * c], cam.rot[3 * c + 1], cam.rot[3 * c + 2]);
    jw[3 + c] = dot3(dm, 0.0, j11, j12, cam.rot[3 * c], cam.rot[3 * c + 1], cam.rot[3 * c + 2]);
  }
  // cov2 = (jw @ cov3) @ jw.T
  double tmp[6];
#pragma unroll
  for (int rr = 0; rr < 2; ++rr)
#pragma unroll
    for (int c = 0; c < 3; ++c)
      tmp[3 * rr + c] = dot3(dm, jw[3 * rr], jw[3 * rr + 1], jw[3 * rr + 2], cov3[c], cov3[3 + c],
                             cov3[6 + c]);
  const double c00 = dot3(dm, tmp[0], tmp[1], tmp[2], jw[0], jw[1], jw[2]);
  const double c01 = dot3(dm, tmp[0], tmp[1], tmp[2], jw[3], jw[4], jw[5]);
  const double c11 = dot3(dm, tmp[3], tmp[4], tmp[5], jw[3], jw[4], jw[5]);
  const double a = c00 + kLowPass, b = c01, c = c11 + kLowPass;
  const double det = a * c - b * b;
  const double mid = 0.5 * (a + c);
  const double amc = a - c;
  const double lam = mid + sqrt(fmax(0.25 * (amc * amc) + b * b, 0.0));
  const double rad = kExtentSigma * sqrt(fmax(lam, 0.0));
  const double cx = (f * tx) / tz + cam.half_w;
  const double cy = (f * ty) / tz + cam.half_h;
  const double x0 = fmax(floor((cx - rad) - 0.5), 0.0);
  const double x1 = fmin(ceil((cx + rad) + 0.5), (double)cam.width);
  const double y0 = fmax(floor((cy - rad) - 0.5), 0.0);
  const double y1 = fmin(ceil((cy + rad) + 0.5), (double)cam.height);
  o.kept = det >= kMinDet && x1 > x0 && y1 > y0;
  o.cx = cx;
  o.cy = cy;
  o.ca = c / det;
  o.cb = -b / det;
  o.cc = a / det;
  if (!o.kept) return;
  o.x0 = (int)x0;
  o.x1 = (int)x1;
  o.y0 = (int)y0;
  o.y1 = (int)y1;
  // evaluate_sh with the world-space view direction (render.py:212-215)
  const double nrm = sqrt((d0 * d0 + d1 * d1) + d2 * d2);
  const double dv = nrm > 0.0 ? nrm : 1.0;
  sh_rgb(r + 11, d0 / dv, d1 / dv, d2 / dv, o.col);
}

// Bulk async copy (TMA engine, 1D) + mbarrier helpers.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

constexpr int kPreStages = 2;
constexpr uint32_t kChunkFloats = kChunkRecords * kRecordFloats;

// Persistent CTAs walk the chunk table (chunk c, c + grid, ...).  Each
// chunk's rows (<= 128 x 236 B, contiguous in the pool) are brought into
// shared memory by one bulk async copy (TMA) while the previous chunk is
// projected, double-buffered on two mbarriers; the per-thread column reads
// of the 59-word records (odd stride) are bank-conflict free.  Chunks whose
// bytes are not 16-byte aligned fall back to plain loads (not the case for
// power-of-two page sizes).
__global__ void __launch_bounds__(kChunkRecords) preprocess_k(
    const float* __restrict__ pool, const Chunk* __restrict__ chunks,
    const FrameDev* __restrict__ fd, uint32_t* __restrict__ key_g, uint32_t* __restrict__ flag,
    BlendRec* __restrict__ rec, uint2* __restrict__ box) {
  extern __shared__ __align__(128) float sbuf[];  // kPreStages x kChunkFloats
  __shared__ __align__(8) uint64_t bar[kPreStages];
  __shared__ Chunk s_chunk[kPreStages];
  __shared__ int s_tma[kPreStages];
  __shared__ RenderCamera cam;
  pdl_wait();
  const uint32_t n = fd->n_chunks;
  if (blockIdx.x >= n) return;
  const uint32_t t = threadIdx.x;
  if (t == 0) {
    cam = fd->cam;
    for (int k = 0; k < kPreStages; ++k) mbar_init(&bar[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // thread 0: start a chunk (descriptor already loaded) into stage st
  auto issue = [&](const Chunk& ch, int st) {
    s_chunk[st] = ch;
    const uint32_t bytes = ch.count * kRecordFloats * 4u;
    const bool tma = (ch.row & 3u) == 0 && (ch.count & 3u) == 0 && ch.count > 0;
    s_tma[st] = tma;
    if (tma) {
      mbar_arrive_tx(&bar[st], bytes);
      bulk_g2s(sbuf + st * kChunkFloats, pool + (size_t)ch.row * kRecordFloats, bytes, &bar[st]);
    } else {
      mbar_arrive_tx(&bar[st], 0u);
    }
  };
  uint32_t phase = 0;  // bit k: parity of stage k's next completion
  int st = 0;
  // thread 0 keeps the next chunk's descriptor one iteration ahead, so its
  // table load never delays the bulk copy it starts
  Chunk next{};
  if (t == 0) {
    issue(chunks[blockIdx.x], 0);
    if (blockIdx.x + gridDim.x < n) next = chunks[blockIdx.x + gridDim.x];
  }
  for (uint32_t c = blockIdx.x; c < n; c += gridDim.x, st ^= 1) {
    const uint32_t cn = c + gridDim.x;
    if (t == 0 && cn < n) {
      issue(next, st ^ 1);  // stage freed by the barrier ending the last iteration
      if (cn + gridDim.x < n) next = chunks[cn + gridDim.x];
    }
    mbar_wait(&bar[st], (phase >> st) & 1u);
    phase ^= 1u << st;
    const Chunk ch = s_chunk[st];
    float* stage = sbuf + st * kChunkFloats;
    if (!s_tma[st]) {
      const float* src = pool + (size_t)ch.row * kRecordFloats;
      for (uint32_t i = t; i < ch.count * kRecordFloats; i += blockDim.x) stage[i] = __ldg(src + i);
      __syncthreads();
    }
    if (t < ch.count) {
      const uint32_t g = ch.gather + t;
      const float* r = stage + t * kRecordFloats;
      Proj p;
      project_one(r, cam, p, true);
      if (!p.kept) {
        flag[g] = 0u;
        key_g[g] = 0xFFFFFFFFu;
      } else {
        BlendRec o;
        o.cx = __double2float_rn(p.cx);
        o.cy = __double2float_rn(p.cy);
        o.ca = __double2float_rn(p.ca);
        o.cb = __double2float_rn(p.cb);
        o.cc = __double2float_rn(p.cc);
        o.r = __double2float_rn(p.col[0]);
        o.g = __double2float_rn(p.col[1]);
        o.b = __double2float_rn(p.col[2]);
        o.alpha = r[10];
        o.bx = (uint32_t)p.x0 | ((uint32_t)p.x1 << 16);
        o.by = (uint32_t)p.y0 | ((uint32_t)p.y1 << 16);
        o.skip = blend_skip(o.alpha);
        rec[g] = o;
        box[g] = make_uint2(o.bx, o.by);
        flag[g] = 1u;
        key_g[g] = __float_as_uint(__double2float_rn(p.tz));
      }
    }
    __syncthreads();  // this stage is refilled next iteration
  }
}

// project_records / compute_keys drop-ins over a contiguous (n, 59) array.
__global__ void project_k(const float* __restrict__ recs, uint32_t n, RenderCamera cam,
                          double* __restrict__ centers, double* __restrict__ conics,
                          float* __restrict__ colors, int32_t* __restrict__ bounds,
                          uint8_t* __restrict__ kept, uint32_t* __restrict__ keys) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float* r = recs + (size_t)i * kRecordFloats;
  Proj p;
  project_one(r, cam, p, false);
  if (keys) keys[i] = p.live ? __float_as_uint(__double2float_rn(p.tz)) : 0xFFFFFFFFu;
  if (!centers) return;
  kept[i] = p.kept ? 1 : 0;
  if (!p.kept) return;
  centers[2 * i] = p.cx;
  centers[2 * i + 1] = p.cy;
  conics[3 * i] = p.ca;
  conics[3 * i + 1] = p.cb;
  conics[3 * i + 2] = p.cc;
  colors[3 * i] = __double2float_rn(p.col[0]);
  colors[3 * i + 1] = __double2float_rn(p.col[1]);
  colors[3 * i + 2] = __double2float_rn(p.col[2]);
  bounds[4 * i] = p.x0;
  bounds[4 * i + 1] = p.x1;
  bounds[4 * i + 2] = p.y0;
  bounds[4 * i + 3] = p.y1;
}

__global__ void sh_k(const double* __restrict__ coeffs, const double* __restrict__ dirs, uint32_t n,
                     double* __restrict__ out) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  sh_rgb(coeffs + 48 * (size_t)i, dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2], out + 3 * i);
}

}  // namespace

namespace {
constexpr size_t kPreSmem = sizeof(float) * kPreStages * kChunkFloats;
int g_pre_grid = 0;  // persistent grid: SMs x resident CTAs
}  // namespace

int32_t preprocess_init() {
  if (g_pre_grid) return VMS_OK;
  VMS_CUDA(cudaFuncSetAttribute((const void*)preprocess_k,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPreSmem));
  int per = 0, dev = 0, sms = 0;
  VMS_CUDA(cudaGetDevice(&dev));
  VMS_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  VMS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, preprocess_k, kChunkRecords,
                                                         kPreSmem));
  g_pre_grid = std::max(1, sms) * std::max(1, per);
  return VMS_OK;
}

int32_t render_preprocess(const float* pool, const Chunk* chunks, uint32_t max_chunks,
                          const RenderWs& w, cudaStream_t s) {
  if (max_chunks == 0) return VMS_OK;
  if (!g_pre_grid) {
    set_error("render_preprocess: preprocess_init() not called");
    return VMS_ERR_INVALID;
  }
  const uint32_t g = std::min<uint32_t>(max_chunks, (uint32_t)g_pre_grid);
  VMS_CUDA(launch(preprocess_k, g, kChunkRecords, kPreSmem, s, pool, chunks,
                  (const FrameDev*)w.fd, w.key_g, w.flag, w.rec, w.box));
  mark("preprocess", s);
  VMS_LAUNCH_CHECK("render_preprocess");
  return VMS_OK;
}

}  // namespace vms

namespace vms {

int32_t project_records(const float* recs, uint32_t n, const RenderCamera& cam, double* centers,
                        double* conics, float* colors, int32_t* bounds, uint8_t* kept,
                        uint32_t* keys, cudaStream_t s) {
  if (n == 0) return VMS_OK;
  project_k<<<ceil_div<uint32_t>(n, 128), 128, 0, s>>>(recs, n, cam, centers, conics, colors,
                                                       bounds, kept, keys);
  VMS_LAUNCH_CHECK("project_records");
  return VMS_OK;
}

int32_t evaluate_sh(const double* coeffs, const double* dirs, uint32_t n, double* out,
                    cudaStream_t s) {
  if (n == 0) return VMS_OK;
  sh_k<<<ceil_div<uint32_t>(n, 128), 128, 0, s>>>(coeffs, dirs, n, out);
  VMS_LAUNCH_CHECK("evaluate_sh");
  return VMS_OK;
}

}  // namespace vms
