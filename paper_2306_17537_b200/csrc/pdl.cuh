// Programmatic dependent launch for chains of dependent kernels in one stream (device helpers
// and the host launcher).  Every kernel launched through launch_pass must call pdl_wait() before
// its first global-memory access and pdl_trigger_late() as its last statement.
#pragma once
#include <cuda_runtime.h>
#include <stdlib.h>

namespace ie {

#ifndef IE_PDL_LATE
#define IE_PDL_LATE 1  // 0: trigger the dependent pass at CTA start instead of CTA exit (A/B build)
#endif
// Programmatic dependent launch (launch_pass): a pass launched with the PDL attribute may be
// scheduled before the previous pass has finished; every global access of the pass comes after
// pdl_wait(), which returns once the previous grid has completed and its writes are visible (a
// no-op without the attribute).  The trigger that lets the next pass's CTAs be scheduled is issued
// as each CTA finishes (pdl_trigger_late), so they take the SMs the exiting CTAs free.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
#if !IE_PDL_LATE
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
__device__ __forceinline__ void pdl_trigger_late() {
#if IE_PDL_LATE
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

// Launch one operator pass with the programmatic-dependent-launch attribute: the next pass's CTAs
// are scheduled as this pass's CTAs exit (pdl_trigger_late) and wait for its completion in
// pdl_wait, so the pass boundary costs no launch gap.  Measured: c2mod
// apply 0.0345 -> 0.0318 ms, c3h 0.1006 -> 0.0905, c4h 0.3421 -> 0.3297, c5 neutral.  (Triggering
// at CTA start instead measured slower on the large grids: c4h 0.369, c5 +10%.)  IE_PDL=0 turns
// it off.
static inline bool use_pdl() {
  static const int env = [] {
    const char* v = getenv("IE_PDL");
    return v ? atoi(v) : 1;
  }();
  return env != 0;
}
template <typename... Args>
static inline void launch_pass(bool pdl, void (*kernel)(Args...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                        Args... args) {
  if (!pdl) {
    kernel<<<grid, block, smem, s>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, args...);
}

}  // namespace ie
