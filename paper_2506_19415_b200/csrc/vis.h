// Visibility / required-page stage interfaces (internal to the .so).
#pragma once

#include <cuda_runtime.h>
#include <cstddef>
#include <stdint.h>

#include "../../include/vmsplat_b200.h"

namespace vms {

using VisCamera = vms_camera;

struct __align__(16) VisTri {
  double ax, ay, bx, by, cx, cy, iza, izb, izc, area;
  int x0, x1, y0, y1;  // inclusive clamped pixel box; x0 > x1 means empty
  uint32_t id;
  uint32_t pad_;
};
static_assert(sizeof(VisTri) == 112 && offsetof(VisTri, x0) == 80, "VisTri layout");

using VisLod = vms_lod;
using RequiredOut = vms_required_out;
using VisArgs = vms_vis_args;

// Per-frame values the visibility kernels read from device memory (so the
// launch sequence can be captured into a CUDA graph once per resolution).
struct VisFrameDev {
  VisCamera cam;
  VisLod lod;
  vms_dpt_frame dpt;  // the device page table's frame inputs (same H2D copy)
};

size_t vis_ws_bytes(uint32_t n_faces, uint32_t page_count);
// One-time setup (shared-memory limits); outside graph capture.
int32_t vis_init();
VisFrameDev* vis_frame_dev(void* ws, uint32_t n_faces, uint32_t page_count);
// [dev] n_tris, n_req, err, 0 of the last vis_launch
uint32_t* vis_meta_dev(void* ws, uint32_t n_faces, uint32_t page_count);
// Upload a.cam / a.lod into the workspace, then vis_launch.
int32_t vis_frame(const VisArgs& a, cudaStream_t s);
// The kernel sequence only (camera and LOD from the workspace block; a.cam's
// width/height fix the raster grid).
int32_t vis_launch(const VisArgs& a, cudaStream_t s);
int32_t reduce_images(const uint32_t* ids, const double* depth, uint64_t n_px,
                      uint32_t page_count, const uint32_t* link_off, const uint32_t* link_tgt,
                      uint32_t* depth_out, uint8_t* direct_out, uint32_t* err, void* ws,
                      cudaStream_t s);
int32_t raster_triangles(const double* raw, const uint32_t* ids, uint32_t n, uint32_t* id_image,
                         double* invz_image, int w, int h, void* ws, cudaStream_t s);

}  // namespace vms
