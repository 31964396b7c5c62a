// NEXT-1: parameter indirection for OPAQUE kernels through a prelude node.
//
// The consumers are launched as plain direct-pointer kernels (standing in for vendor kernels whose
// code cannot be rewritten) with the device-updatable attribute. The prelude node at the root of
// the graph dereferences the pointer cells (the device pointer table, written by one H2D copy per
// replay) and writes each value into the consumer node's parameter buffer at its byte
// offset with the device graph API cudaGraphKernelNodeSetParam. One thread per patch;
// a gpu-scope fence before the dependents are triggered makes the updates visible to the launches
// that follow (cuda_device_runtime_api.h contract for device node updates + PDL).
//
// Built with relocatable device code (device runtime API), device-linked into libcgx.so.
#include <cuda_runtime.h>
#include <stdint.h>

#include "cgx_device.cuh"
#include "cgx_prelude.h"

namespace cgx {

__global__ void k_prelude(const __grid_constant__ PreludeArgs a) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n_patches; i += gridDim.x * blockDim.x) {
    const PreludePatch p = a.patches[i];
    const uint64_t v = ld_table(a.table + p.ext_j);            // dereference the pointer cell px
    cudaGraphKernelNodeSetParam(p.node, p.offset, &v, sizeof(v));
  }
  __threadfence();
  __syncthreads();
  pdl_trigger();
}

const void* kfn_prelude() { return (const void*)k_prelude; }

// NEXT-4: one replay step of the device-side loop. Replay i = *iter: copy pointer set i % n_sets
// into the table, fence, then tail-launch the chain graph and this scheduler's own graph. Tail
// launches start after the launching graph completes and run one after another in enqueue order,
// so the chain of replay i reads the table after this kernel wrote it, and the next scheduler
// step (which overwrites the table) starts only after that chain has completed.
__global__ void k_devloop(const __grid_constant__ DevLoopArgs a) {
  __shared__ unsigned long long s_i;
  if (threadIdx.x == 0) s_i = *a.iter;
  __syncthreads();
  const unsigned long long i = s_i;
  if (i >= a.n_replays) return;
  const uint64_t* src = a.sets + (size_t)(i % a.n_sets) * a.n_ext;
  for (uint32_t j = threadIdx.x; j < a.n_ext; j += blockDim.x) a.table[j] = src[j];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    *a.iter = i + 1;
    __threadfence();
    // a failed device launch ends the loop and is reported through the exec's status word (the
    // host's next cgx_launch returns CGX_E_DEVICE) instead of trapping the context
    bool ok = cudaGraphLaunch(a.chain, cudaStreamGraphTailLaunch) == cudaSuccess;
    if (ok && i + 1 < a.n_replays)
      ok = cudaGraphLaunch(cudaGetCurrentGraphExec(), cudaStreamGraphTailLaunch) == cudaSuccess;
    if (!ok && a.status)
      asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(a.status), "r"(kDevErrDevLaunch) : "memory");
  }
}

const void* kfn_devloop() { return (const void*)k_devloop; }

}  // namespace cgx
