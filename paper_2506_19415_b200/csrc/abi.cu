// extern "C" boundary of libvmsplat_b200.so (declared in include/vmsplat_b200.h).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>
#include <algorithm>

#include <cstdlib>

#include "common.cuh"
#include "prims.h"
#include "render.h"
#include "vis.h"

namespace vms {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int32_t cuda_status(cudaError_t e, const char* where) {
  set_error("%s: %s", where, cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? VMS_ERR_NOMEM : VMS_ERR_CUDA;
}

bool g_profile = false;

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("VMSPLAT_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
namespace {
struct Mark {
  const char* name;
  cudaStream_t stream;
  cudaEvent_t ev;
};
std::vector<Mark> g_marks;
std::vector<cudaEvent_t> g_event_pool;
size_t g_pool_used = 0;
}  // namespace

void mark_impl(const char* name, cudaStream_t s) {
  if (g_pool_used == g_event_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    g_event_pool.push_back(e);
  }
  cudaEvent_t e = g_event_pool[g_pool_used++];
  cudaEventRecord(e, s);
  g_marks.push_back({name, s, e});
}

namespace {

template <typename T>
T* carve(char*& p, size_t n) {
  uintptr_t a = (reinterpret_cast<uintptr_t>(p) + 255) & ~uintptr_t(255);
  T* r = reinterpret_cast<T*>(a);
  p = reinterpret_cast<char*>(a + sizeof(T) * n);
  return r;
}

__global__ void iota_k(uint32_t* v, uint32_t n) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}

__global__ void gather_i64_k(const int64_t* src, const uint32_t* perm, int64_t* dst, uint32_t n) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[perm[i]];
}

__global__ void world_to_view_k(const double* __restrict__ p, int64_t n, vms_camera cam,
                                double* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double d0 = __dsub_rn(p[3 * i], cam.pos[0]);
  const double d1 = __dsub_rn(p[3 * i + 1], cam.pos[1]);
  const double d2 = __dsub_rn(p[3 * i + 2], cam.pos[2]);
#pragma unroll
  for (int j = 0; j < 3; ++j)
    out[3 * i + j] = dot3(cam.dot_mode, d0, d1, d2, cam.rot[j], cam.rot[3 + j], cam.rot[6 + j]);
}

// Page upload through mapped pinned host memory: one launch for the whole
// plan, 16-byte loads over PCIe when every copy is 16-byte aligned.
__global__ void upload_k(const vms_copy* __restrict__ copies, int64_t n,
                         const char* __restrict__ host, char* __restrict__ dev, int vec16) {
  for (int64_t c = blockIdx.y; c < n; c += gridDim.y) {
    const vms_copy cp = copies[c];
    const char* s = host + cp.src_offset;
    char* d = dev + cp.dst_offset;
    if (vec16) {
      const uint64_t n16 = cp.nbytes / 16;
      const uint4* s4 = reinterpret_cast<const uint4*>(s);
      uint4* d4 = reinterpret_cast<uint4*>(d);
      for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n16;
           i += (uint64_t)gridDim.x * blockDim.x)
        d4[i] = s4[i];
    } else {
      const uint64_t n4 = cp.nbytes / 4;
      const uint32_t* s1 = reinterpret_cast<const uint32_t*>(s);
      uint32_t* d1 = reinterpret_cast<uint32_t*>(d);
      for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4;
           i += (uint64_t)gridDim.x * blockDim.x)
        d1[i] = s1[i];
    }
  }
}

}  // namespace
}  // namespace vms

using namespace vms;

extern "C" {

const char* vms_last_error(void) { return g_err; }

int32_t vms_profile_enable(int32_t on) {
  g_profile = on != 0;
  g_marks.clear();
  g_pool_used = 0;
  return VMS_OK;
}

int64_t vms_profile_report(char* buf, int64_t len) {
  // per kernel name: count and summed device time (us) between a mark and the
  // previous mark on the same stream ("begin" marks open a sequence)
  std::vector<std::pair<std::string, std::pair<int64_t, double>>> agg;
  std::map<cudaStream_t, cudaEvent_t> last;
  for (const Mark& m : g_marks) {
    cudaEventSynchronize(m.ev);
    auto it = last.find(m.stream);
    if (it != last.end() && std::strcmp(m.name, "begin") != 0) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, it->second, m.ev);
      size_t k = 0;
      while (k < agg.size() && agg[k].first != m.name) ++k;
      if (k == agg.size()) agg.push_back({m.name, {0, 0.0}});
      agg[k].second.first += 1;
      agg[k].second.second += 1e3 * ms;
    }
    last[m.stream] = m.ev;
  }
  std::string out;
  char line[256];
  for (auto& a : agg) {
    snprintf(line, sizeof(line), "%s,%lld,%.3f\n", a.first.c_str(), (long long)a.second.first,
             a.second.second);
    out += line;
  }
  if (buf && len > 0) {
    const size_t n = std::min<size_t>(out.size(), (size_t)len - 1);
    std::memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return (int64_t)out.size();
}

int32_t vms_abi_version(void) { return VMS_ABI_VERSION; }

int32_t vms_tile_size(void) { return tile_size(); }

int32_t vms_debug_blend_trace(void* dev_ptr) { return debug_blend_trace(dev_ptr); }

int32_t vms_debug_cert_all(int32_t on) { return debug_cert_all(on); }
int32_t vms_debug_lane_lists(int32_t on, int32_t margin) { return debug_lane_lists(on, margin); }

int32_t vms_debug_exp(const double* x, int64_t n, double* out, void* stream) {
  if (n < 0 || (n > 0 && (!x || !out))) {
    set_error("debug_exp: bad arguments");
    return VMS_ERR_INVALID;
  }
  return debug_exp(x, (uint64_t)n, out, static_cast<cudaStream_t>(stream));
}

int32_t vms_host_accessible(const void* ptr) {
  if (!ptr) return 0;
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return at.type == cudaMemoryTypeHost && at.devicePointer == ptr ? 1 : 0;
}

int32_t vms_host_register(const void* ptr, uint64_t bytes, int32_t read_only, void** base_out) {
  // page-align the range: the record section of a memory-mapped .vms file
  // starts at a section offset, not on a page boundary
  if (!ptr || !bytes || !base_out) {
    set_error("host_register: null pointer or empty range");
    return VMS_ERR_INVALID;
  }
  const uintptr_t pg = 4096;
  const uintptr_t a = (uintptr_t)ptr & ~(pg - 1);
  const uintptr_t b = ((uintptr_t)ptr + bytes + pg - 1) & ~(pg - 1);
  unsigned flags = cudaHostRegisterPortable | cudaHostRegisterMapped;
  if (read_only) flags |= cudaHostRegisterReadOnly;
  cudaError_t e = cudaHostRegister((void*)a, (size_t)(b - a), flags);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return cuda_status(e, "cudaHostRegister");
  }
  *base_out = (void*)a;
  return VMS_OK;
}

int32_t vms_host_unregister(void* base) {
  if (!base) return VMS_OK;
  cudaError_t e = cudaHostUnregister(base);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return cuda_status(e, "cudaHostUnregister");
  }
  return VMS_OK;
}

size_t vms_composite_workspace_bytes(int64_t n, int64_t n_instances, int32_t h, int32_t w) {
  const uint32_t tiles = tile_count(w, h);
  return render_ws_bytes((uint32_t)(n > 0 ? n : 1),
                         (uint32_t)(n_instances > 0 ? n_instances : 1), tiles);
}

int32_t vms_composite_splats(const float* centers, const float* conics, const float* colors,
                             const float* alphas, const int32_t* bounds, int64_t n,
                             int64_t n_instances, float* image, int32_t h, int32_t w,
                             int32_t exact, void* workspace, size_t workspace_bytes,
                             void* stream) {
  if (n < 0 || n_instances < 0 || n_instances > 0xFFFFFFFFll || h < 1 || w < 1 || !image || (n > 0 && (!centers || !conics || !colors ||
                                                       !alphas || !bounds))) {
    set_error("composite_splats: invalid arguments");
    return VMS_ERR_INVALID;
  }
  if (workspace_bytes < vms_composite_workspace_bytes(n, n_instances, h, w)) {
    set_error("composite_splats: workspace too small");
    return VMS_ERR_INVALID;
  }
  int32_t rc0 = blend_init();
  if (rc0) return rc0;
  const uint32_t tiles = tile_count(w, h);
  RenderWs ws = render_carve(workspace, (uint32_t)(n > 0 ? n : 1),
                             (uint32_t)(n_instances > 0 ? n_instances : 1), tiles);
  return composite_ordered(centers, conics, colors, alphas, bounds, (uint32_t)n, image, h, w,
                           exact, ws, static_cast<cudaStream_t>(stream));
}

size_t vms_rasterize_workspace_bytes(int64_t n) { return sizeof(VisTri) * (size_t)(n + 1); }

int32_t vms_rasterize_triangles(const double* tris, const uint32_t* ids, int64_t n,
                                uint32_t* id_image, double* invz_image, int32_t h, int32_t w,
                                void* workspace, size_t workspace_bytes, void* stream) {
  if (n < 0 || h < 1 || w < 1 || !id_image || !invz_image || (n > 0 && (!tris || !ids))) {
    set_error("rasterize_triangles: invalid arguments");
    return VMS_ERR_INVALID;
  }
  if (workspace_bytes < vms_rasterize_workspace_bytes(n)) {
    set_error("rasterize_triangles: workspace too small");
    return VMS_ERR_INVALID;
  }
  return raster_triangles(tris, ids, (uint32_t)n, id_image, invz_image, w, h, workspace,
                          static_cast<cudaStream_t>(stream));
}

size_t vms_radix_workspace_bytes(int64_t n) {
  const size_t m = (size_t)(n > 0 ? n : 1);
  return sizeof(uint32_t) * m * 4 + sizeof(int64_t) * m + radix_ws_bytes((uint32_t)m) + 256 * 8;
}

int32_t vms_radix_sort_pairs(uint32_t* keys, int64_t* values, int64_t n, void* workspace,
                             size_t workspace_bytes, void* stream) {
  if (n < 0 || n > 0xFFFFFFFFll || (n > 0 && (!keys || !values))) {
    set_error("radix_sort_pairs: invalid arguments");
    return VMS_ERR_INVALID;
  }
  if (workspace_bytes < vms_radix_workspace_bytes(n)) {
    set_error("radix_sort_pairs: workspace too small");
    return VMS_ERR_INVALID;
  }
  if (n == 0) return VMS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* p = static_cast<char*>(workspace);
  const uint32_t m = (uint32_t)n;
  uint32_t* k0 = carve<uint32_t>(p, m);
  uint32_t* v0 = carve<uint32_t>(p, m);
  uint32_t* k1 = carve<uint32_t>(p, m);
  uint32_t* v1 = carve<uint32_t>(p, m);
  int64_t* tmp = carve<int64_t>(p, m);
  void* rws = carve<char>(p, radix_ws_bytes(m));
  VMS_CUDA(cudaMemcpyAsync(k0, keys, sizeof(uint32_t) * m, cudaMemcpyDeviceToDevice, s));
  iota_k<<<ceil_div<uint32_t>(m, 256), 256, 0, s>>>(v0, m);
  int alt = 0;
  int32_t st = radix_sort_u32(k0, v0, k1, v1, nullptr, m, m, 0, 32, &alt, rws, s);
  if (st) return st;
  uint32_t* ks = alt ? k1 : k0;
  uint32_t* vs = alt ? v1 : v0;
  gather_i64_k<<<ceil_div<uint32_t>(m, 256), 256, 0, s>>>(values, vs, tmp, m);
  VMS_CUDA(cudaMemcpyAsync(keys, ks, sizeof(uint32_t) * m, cudaMemcpyDeviceToDevice, s));
  VMS_CUDA(cudaMemcpyAsync(values, tmp, sizeof(int64_t) * m, cudaMemcpyDeviceToDevice, s));
  VMS_LAUNCH_CHECK("radix_sort_pairs");
  return VMS_OK;
}

int32_t vms_world_to_view(const double* points, int64_t n, const vms_camera* cam, double* out,
                          void* stream) {
  if (n < 0 || !cam || (n > 0 && (!points || !out))) {
    set_error("world_to_view: invalid arguments");
    return VMS_ERR_INVALID;
  }
  if (n == 0) return VMS_OK;
  world_to_view_k<<<(unsigned)ceil_div<int64_t>(n, 256), 256, 0,
                    static_cast<cudaStream_t>(stream)>>>(points, n, *cam, out);
  VMS_LAUNCH_CHECK("world_to_view");
  return VMS_OK;
}

int32_t vms_project_records(const float* records, int64_t n, const vms_camera* cam,
                            double* centers, double* conics, float* colors, int32_t* bounds,
                            uint8_t* kept, uint32_t* keys, void* stream) {
  const bool geo = centers || conics || colors || bounds || kept;
  if (n < 0 || n > 0xFFFFFFFFll || !cam || (n > 0 && !records) ||
      (geo && !(centers && conics && colors && bounds && kept))) {
    set_error("project_records: invalid arguments");
    return VMS_ERR_INVALID;
  }
  return project_records(records, (uint32_t)n, *cam, centers, conics, colors, bounds, kept, keys,
                         static_cast<cudaStream_t>(stream));
}

int32_t vms_evaluate_sh(const double* coeffs, const double* dirs, int64_t n, double* out,
                        void* stream) {
  if (n < 0 || n > 0xFFFFFFFFll || (n > 0 && (!coeffs || !dirs || !out))) {
    set_error("evaluate_sh: invalid arguments");
    return VMS_ERR_INVALID;
  }
  return evaluate_sh(coeffs, dirs, (uint32_t)n, out, static_cast<cudaStream_t>(stream));
}

size_t vms_visibility_workspace_bytes(uint32_t n_faces, uint32_t page_count) {
  return vis_ws_bytes(n_faces, page_count);
}

int32_t vms_visibility(const vms_vis_args* args, void* stream) {
  if (!args || !args->workspace || args->cam.width < 1 || args->cam.height < 1 ||
      args->lod.count < 0 || args->lod.count > 8) {
    set_error("visibility: invalid arguments");
    return VMS_ERR_INVALID;
  }
  return vis_frame(*args, static_cast<cudaStream_t>(stream));
}

int32_t vms_reduce_visibility(const uint32_t* page_image, const double* depth_image,
                              int64_t n_pixels, uint32_t page_count, const uint32_t* link_off,
                              const uint32_t* link_tgt, uint32_t* depths_out, uint8_t* direct_out,
                              uint32_t* bad_id_out, void* workspace, size_t workspace_bytes,
                              void* stream) {
  if (n_pixels < 0 || !depths_out || !direct_out || !bad_id_out || !link_off ||
      (n_pixels > 0 && (!page_image || !depth_image)) ||
      workspace_bytes < sizeof(uint32_t) * ((size_t)page_count + 1)) {
    set_error("reduce_visibility: invalid arguments");
    return VMS_ERR_INVALID;
  }
  return reduce_images(page_image, depth_image, (uint64_t)n_pixels, page_count, link_off,
                       link_tgt, depths_out, direct_out, bad_id_out, workspace,
                       static_cast<cudaStream_t>(stream));
}

int32_t vms_upload_pages(const vms_copy* copies, int64_t n, const void* host_base,
                         void* dev_base, int32_t mode, void* stream) {
  if (n < 0 || (n > 0 && (!copies || !host_base || !dev_base))) {
    set_error("upload_pages: invalid arguments");
    return VMS_ERR_INVALID;
  }
  if (n == 0) return VMS_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (mode == 0) {
    // copy engines: one cudaMemcpyAsync per run of copies that are adjacent
    // in both the host scene and the destination (no SM time - the pages
    // stream in while the previous frame renders at full SM occupancy)
    const char* h = static_cast<const char*>(host_base);
    char* d = static_cast<char*>(dev_base);
    int64_t i = 0;
    while (i < n) {
      uint64_t src = copies[i].src_offset, dst = copies[i].dst_offset, nb = copies[i].nbytes;
      int64_t j = i + 1;
      while (j < n && copies[j].src_offset == src + nb && copies[j].dst_offset == dst + nb) {
        nb += copies[j].nbytes;
        ++j;
      }
      VMS_CUDA(cudaMemcpyAsync(d + dst, h + src, nb, cudaMemcpyHostToDevice, s));
      i = j;
    }
    return VMS_OK;
  }
  mark("begin", s);
  // 16-byte vector copies only when the bases are aligned too: a scene
  // registered in place is the file mapping plus the header, not 16-aligned
  int vec16 = ((reinterpret_cast<uintptr_t>(host_base) | reinterpret_cast<uintptr_t>(dev_base)) &
               15u) == 0;
  for (int64_t i = 0; i < n; ++i)
    vec16 &= ((copies[i].src_offset | copies[i].dst_offset | copies[i].nbytes) & 15u) == 0;
  dim3 grid(64, (unsigned)(n < 65535 ? n : 65535));
  upload_k<<<grid, 256, 0, s>>>(copies, n, static_cast<const char*>(host_base),
                                static_cast<char*>(dev_base), vec16);
  mark("upload", s);
  VMS_LAUNCH_CHECK("upload_pages");
  return VMS_OK;
}

size_t vms_render_workspace_bytes(uint32_t n_cap, uint32_t m_cap, int32_t width,
                                  int32_t height) {
  const uint32_t tiles = tile_count(width, height);
  return render_ws_bytes(n_cap, m_cap, tiles);
}

int32_t vms_render(const vms_render_args* a, void* stream) {
  if (!a || !a->workspace || !a->image || a->cam.width < 1 || a->cam.height < 1 ||
      a->n_splats > a->n_cap || (a->n_chunks && (!a->pool || !a->chunks))) {
    set_error("render: invalid arguments");
    return VMS_ERR_INVALID;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int32_t rc0 = blend_init();
  if (rc0) return rc0;
  const uint32_t tiles =
      tile_count(a->cam.width, a->cam.height);
  RenderWs w = render_carve(a->workspace, a->n_cap, a->m_cap, tiles);
  mark("begin", s);
  FrameDev f{};
  f.cam = a->cam;
  f.image = a->image;
  f.n_chunks = a->n_chunks;
  f.n_splats = a->n_splats;
  int32_t st = render_upload_frame(w, f, s);
  if (st) return st;
  st = render_clear(a->cam.width, a->cam.height, w, s);
  if (st) return st;
  st = render_preprocess(a->pool, a->chunks, a->n_chunks, w, s);
  if (st) return st;
  if (a->events[0]) VMS_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(a->events[0]), s));
  st = render_finish(a->cam.width, a->cam.height, w, a->accumulate, a->exact, a->events, false, 1,
                     s);
  if (st) return st;
  if (a->counters_out)
    VMS_CUDA(cudaMemcpyAsync(a->counters_out, w.ctr, sizeof(uint32_t) * 4,
                             cudaMemcpyDeviceToHost, s));
  return VMS_OK;
}

}  // extern "C"
