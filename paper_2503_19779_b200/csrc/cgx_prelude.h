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

}  // namespace cgx
