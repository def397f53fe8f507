// Splat-render stage interfaces (internal to the .so): preprocess over the
// resident page chunks, depth sort, tile duplication, tile sort, blend.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/vmsplat_b200.h"

namespace vms {

constexpr int kRecordFloats = 59;   // gaussians.py:1-33
constexpr int kChunkRecords = 128;  // records per preprocess CTA
// Blend tile edge in pixels (32 by default; VMSPLAT_TILE=16 selects 16x16).
int tile_size();
uint32_t tile_count(int width, int height);

using RenderCamera = vms_camera;
using Chunk = vms_chunk;

// Per-splat blend payload, 48 B (3 x 16 B): f32 center/conic exactly as the
// reference wrapper casts them (kernels/__init__.py:27-28), f32 colour
// (render.py:215), f32 alpha, half-open int16 pixel bounds.
struct __align__(16) BlendRec {
  float cx, cy;
  float ca, cb, cc;
  float r, g, b;
  float alpha;
  uint32_t bx;  // x0 | x1 << 16
  uint32_t by;  // y0 | y1 << 16
  float skip;   // f32 <= log(2^-36 / alpha): sigma below it cannot change f32 T
};

// Exp-skip threshold of a splat, rounded down so that skipping is always
// conservative (alpha * exp(sigma) < 2^-36 for sigma < skip).
__device__ __forceinline__ float blend_skip(float alpha) {
  return alpha > 0.f ? __double2float_rd(log(0x1p-36 / (double)alpha)) : -3.0e38f;
}

// Per-frame values every render kernel reads from device memory, so that a
// frame's launch sequence is identical from frame to frame and can be
// captured once into a CUDA graph (the host uploads this block, the chunk
// table and the page copies before each graph launch).
struct FrameDev {
  vms_camera cam;
  float* image;       // (h, w, 3) f32 output of this frame
  uint32_t n_chunks;  // chunk-table rows in use
  uint32_t n_splats;  // gather indices in use (resident records)
  // optional host-mapped copy of the counters (n_kept, n_inst, overflow,
  // n_need), written by tile_prep_k: no copy-engine transfer queued behind
  // a previous frame's image copy on the main stream
  uint32_t* counters_host;
};

// Frame counters living in device memory.
struct RenderCounters {
  uint32_t n_kept;
  uint32_t n_inst;
  uint32_t overflow;
  uint32_t n_need;  // instances the frame needs (== n_inst unless overflow)
};

struct RenderWs {
  uint32_t n_cap;  // splat capacity (gather indices)
  uint32_t m_cap;  // tile-instance capacity
  uint32_t *key_g, *flag, *pos;
  BlendRec* rec;
  uint2* box;      // the records' packed (bx, by) box words, for dup_count_k
  uint32_t *k0, *v0, *k1, *v1;
  uint32_t *cnt, *off;
  uint32_t *tk0, *tv0, *tk1, *tv1;
  uint32_t* rects;   // packed tile rectangle per sorted splat
  uint32_t* tcount;  // instances per tile
  uint32_t* tdiff;   // 2D difference array of tcount ((tiles_x + 1) x (tiles_y + 1))
  uint32_t* ranges;  // 2 per tile
  uint32_t* order;   // blend schedule: tiles, longest list first
  uint32_t* hot;     // [0] hot tiles this frame, [1..] their ids (blend_hot_k)
  uint32_t* tile_hot;  // per tile: 1 if blend_hot_k owns it
  uint32_t* cert;      // certified fast blend: flagged-pixel count per band
  uint4* cert_list;    // {pixel, initial r, g, b bits} per flagged pixel, by band
  RenderCounters* ctr;
  FrameDev* fd;
  void* scan_ws;
  void* scan_ws2;  // the second scan of a frame (tile instance offsets)
  void* radix_ws;
};

size_t render_ws_bytes(uint32_t n_cap, uint32_t m_cap, uint32_t n_tiles);
RenderWs render_carve(void* ws, uint32_t n_cap, uint32_t m_cap, uint32_t n_tiles);

// Preprocess (EWA + SH, FP64) of every record named by the chunk table;
// writes key_g / flag / rec at gather indices.  Camera and chunk count come
// from w.fd; max_chunks bounds the grid (CTAs past fd->n_chunks exit).
int32_t render_preprocess(const float* pool, const Chunk* chunks, uint32_t max_chunks,
                          const RenderWs& w, cudaStream_t s);

// From preprocessed splats to an image: compaction, depth sort, tile
// duplication, tile sort, ranges, blend.  Splat count and image pointer come
// from w.fd; width/height fix the tile grid.  `events` (optional, 4) are
// recorded after preprocess-side stages; `external` marks them as graph
// event-record nodes when the sequence is being captured.
// `bands` > 1 splits the blend into that many launches over horizontal
// bands of tile rows; bands < 0 builds the schedule for -bands bands and
// stops there: the caller launches the bands itself with render_band (e.g.
// to start each band's device->host copy as soon as it is blended).
int32_t render_finish(int width, int height, const RenderWs& w, int accumulate, int exact,
                      void* const* events, bool external, int bands, cudaStream_t s);
int32_t render_band(int width, int height, const RenderWs& w, int exact, int band, int bands,
                    cudaStream_t s);
int blend_band_row(int b, int bands, int tiles_y);

// One-time setup (constant tables, shared-memory limits, persistent grid
// sizes); must run before the first render launch and outside graph capture.
// blend_init() also runs preprocess_init().
int32_t blend_init();
int32_t preprocess_init();

// Per-CTA blend timing trace (profiling only; nullptr disables).
int32_t debug_blend_trace(void* dev_ptr);
int32_t debug_exp(const double* x, uint64_t n, double* out, cudaStream_t s);
// Certified fast blend: flag every pixel (tests); pixels flagged by the
// last blend (synchronises the device).
int32_t debug_cert_all(int on);
// exact blend: lane lists on/off and their step margin (tests, A/B)
int32_t debug_lane_lists(int on, int margin);
int32_t debug_cert_count(const RenderWs& w, uint32_t* out);

// Zero the frame's counters and primitive workspaces (all memsets of a
// frame, ahead of its first kernel); render_finish assumes it ran.
int32_t render_clear(int width, int height, const RenderWs& w, cudaStream_t s);

// Stage FrameDev from host memory (pageable or pinned) into w.fd.
int32_t render_upload_frame(const RenderWs& w, const FrameDev& f, cudaStream_t s);

// project_records / compute_keys over a contiguous record array; any output
// pointer may be null except that centers..kept come together.
int32_t project_records(const float* recs, uint32_t n, const RenderCamera& cam, double* centers,
                        double* conics, float* colors, int32_t* bounds, uint8_t* kept,
                        uint32_t* keys, cudaStream_t s);
int32_t evaluate_sh(const double* coeffs, const double* dirs, uint32_t n, double* out,
                    cudaStream_t s);

// Kernel-level composite of caller-ordered splats (composite_splats).
int32_t composite_ordered(const float* centers, const float* conics, const float* colors,
                          const float* alphas, const int32_t* bounds, uint32_t n, float* image,
                          int h, int w, int exact, const RenderWs& ws, cudaStream_t s);

}  // namespace vms
