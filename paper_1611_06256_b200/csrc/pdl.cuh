// pdl.cuh -- programmatic dependent launch.  Every kernel of the hot path is
// launched with cudaLaunchAttributeProgrammaticStreamSerialization, signals
// griddepcontrol.launch_dependents once its own setup is done, and executes
// griddepcontrol.wait before its first global-memory access.  The next
// kernel's CTAs therefore launch and run their prologue (TMEM allocation,
// mbarrier init, address tables) while the previous kernel drains; the wait
// still orders every read and write after the predecessor's completion, so
// results are unchanged.  Both instructions are no-ops without the attribute.
#pragma once

namespace ga3c {

__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Both, for kernels with no setup worth overlapping.
__device__ __forceinline__ void pdl_enter() {
  pdl_trigger();
  pdl_wait();
}

}  // namespace ga3c
