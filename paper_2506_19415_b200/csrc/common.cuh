// Shared device helpers for the vmsplat B200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/vmsplat_b200.h"

#define VMS_DEV __device__ __forceinline__

namespace vms {

constexpr int kWarp = 32;
constexpr int kSMs = 148;

// Thread-local last error string (filled by the ABI layer).
void set_error(const char* fmt, ...);
int32_t cuda_status(cudaError_t e, const char* where);

// Optional per-launch device timing (vms_profile_enable): records a CUDA
// event after each kernel; vms_profile_report turns consecutive events on a
// stream into per-kernel device times.  A no-op unless enabled.
extern bool g_profile;
void mark_impl(const char* name, cudaStream_t s);
inline void mark(const char* name, cudaStream_t s) {
  if (g_profile) mark_impl(name, s);
}

#define VMS_CUDA(call)                                         \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return ::vms::cuda_status(_e, #call); \
  } while (0)

#define VMS_LAUNCH_CHECK(where)                                 \
  do {                                                          \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e != cudaSuccess) return ::vms::cuda_status(_e, where); \
  } while (0)

VMS_DEV uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

VMS_DEV int lane_id() { return threadIdx.x & 31; }

// Non-contracted FP64 helpers: the exactness-critical stages follow NumPy's
// elementwise semantics (no FMA) and OpenBLAS's fused dot order explicitly.
VMS_DEV double dmul(double a, double b) { return __dmul_rn(a, b); }
VMS_DEV double dadd(double a, double b) { return __dadd_rn(a, b); }
VMS_DEV double dsub(double a, double b) { return __dsub_rn(a, b); }
VMS_DEV double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// 3-term dot product in the order the host BLAS uses (probed at session
// start): mode 0 = fma(a2,b2, fma(a1,b1, a0*b0)),
// mode 1 = (a0*b0 + a1*b1) + a2*b2 without contraction.
VMS_DEV double dot3(int mode, double a0, double a1, double a2, double b0, double b1,
                    double b2) {
  if (mode == 0) return __fma_rn(a2, b2, __fma_rn(a1, b1, __dmul_rn(a0, b0)));
  return __dadd_rn(__dadd_rn(__dmul_rn(a0, b0), __dmul_rn(a1, b1)), __dmul_rn(a2, b2));
}

// Programmatic dependent launch (sm_90+): the kernels of the frame graphs
// are launched with programmatic stream serialization, so a kernel's CTAs
// are scheduled while its predecessor drains; each kernel calls pdl_wait()
// before it touches anything an earlier kernel wrote (it returns once the
// predecessor grid has completed and its writes are visible - and the
// predecessor itself waited, so the chain is transitive).  Without the
// launch attribute the wait is a no-op.  VMSPLAT_PDL=0 disables it.
VMS_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();

template <typename... KArgs, typename... Args>
cudaError_t launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                   cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <typename T>
__host__ __device__ __forceinline__ T ceil_div(T a, T b) {
  return (a + b - 1) / b;
}

}  // namespace vms
