// NEXT-1 prelude-kernel parameter indirection (see k_prelude.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cgx {

struct PreludePatch {
  cudaGraphDeviceNode_t node;   // device-updatable consumer node
  uint32_t offset;              // byte offset of the pointer in its parameter buffer
  uint32_t ext_j;               // pointer cell (table index)
};

struct PreludeArgs {
  const uint64_t* table;        // pointer cells px_j, written by one H2D copy per replay
  const PreludePatch* patches;  // device array
  uint32_t n_patches;
  uint32_t pad;
};

const void* kfn_prelude();

// NEXT-4 device-side replay loop (k_prelude.cu, k_devloop)
struct DevLoopArgs {
  uint64_t* table;              // the exec's pointer table
  const uint64_t* sets;         // [n_sets][n_ext] pointer sets (device)
  unsigned long long* iter;     // replays started so far (device counter, reset per loop)
  unsigned long long n_replays;
  cudaGraphExec_t chain;        // device-launchable chain graph
  uint32_t n_ext, n_sets;
  uint32_t* status;             // exec status word (mapped host memory): kDevErrDevLaunch
};
const void* kfn_devloop();

}  // namespace cgx
