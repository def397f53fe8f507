// Device-wide primitives whose element counts may live in device memory
// (the per-frame counts - clipped triangles, kept splats, tile instances -
// are produced on the GPU and never read back mid-frame).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace vms {

// Exclusive scan of n u32 values; n = *n_dev when n_dev != nullptr, else
// n_host.  *total (device, optional) receives the sum.  ws needs
// scan_ws_bytes() bytes.
// n_max: upper bound on n (sizes the look-back status array in ws).
size_t scan_ws_bytes(uint32_t n_max);
// clear = false: the caller zeroed the first scan_ws_bytes(n_max) of ws
// (e.g. hoisted to the start of a captured frame, so the kernels chain).
int32_t scan_exclusive_u32(const uint32_t* in, uint32_t* out, const uint32_t* n_dev,
                           uint32_t n_host, uint32_t n_max, uint32_t* total, void* ws,
                           cudaStream_t s, bool clear = true);

// Stable LSD radix sort of (u32 key, u32 value) pairs over key bits
// [begin_bit, end_bit).  Ping-pongs between (k0,v0) and (k1,v1); returns via
// *in_alt whether the sorted result ended in (k1, v1).  n as for the scan.
// clear = false: the caller zeroed the first radix_clear_bytes() of ws.
size_t radix_ws_bytes(uint32_t n_max);
size_t radix_clear_bytes();
int32_t radix_sort_u32(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1,
                       const uint32_t* n_dev, uint32_t n_host, uint32_t n_max, int begin_bit,
                       int end_bit, int* in_alt, void* ws, cudaStream_t s, bool clear = true);

// The same sort for callers that produce the digit histograms themselves
// (e.g. from per-bin counts they already have).  Before the call: counters
// zero, ghist[p][d] = count of digit d in pass p, and for every pass the
// first ceil(n / tile_items) * 256 status words zero.  n comes from n_dev.
struct RadixLayout {
  uint32_t* counters;  // [64]
  uint32_t* ghist;     // [4][256]
  uint32_t* status;    // [pass][pass_stride]
  size_t pass_stride;
  uint32_t tile_items;
};
RadixLayout radix_layout(void* ws, uint32_t n_max);
int32_t radix_passes_u32(uint32_t* k0, uint32_t* v0, uint32_t* k1, uint32_t* v1,
                         const uint32_t* n_dev, uint32_t n_max, int begin_bit, int end_bit,
                         int* in_alt, void* ws, cudaStream_t s);

}  // namespace vms
