// Device-side helpers for sm_100a: programmatic dependent launch, cache-hinted loads/stores.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "cgx_args.h"

namespace cgx {

// T5 first node: CTA 0 publishes the by-value pointer array into the device table, then makes the
// stores visible at gpu scope (fence) before any of its threads triggers the dependents. The next
// node is launched only after every CTA of this one has triggered, so its pre-wait table fetch
// (an L2 load) observes the published pointers. Called before the kernel's own trigger.
template <typename Base, int CAP>
__device__ __forceinline__ void tw_publish(const ArgsTW<Base, CAP>& A) {
  if constexpr (CAP > 0) {
    if (blockIdx.x == 0) {
      for (uint32_t i = threadIdx.x; i < A.tw.n; i += blockDim.x) A.tw.table[i] = A.tw.ptr[i];
      __threadfence();
      __syncthreads();
    }
  }
}

// Programmatic dependent launch (PDL). A kernel's prologue (pointer-table fetch, loads of slots
// nothing in the graph writes) may run while its predecessors drain; everything that reads another
// node's output comes after pdl_wait(). See the protocol note in cgx_args.h.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

__device__ __forceinline__ unsigned long long gtimer();
// Bounded spin (DevStatus, cgx_args.h): call once per poll with the poll start time; every 1024
// polls the elapsed %globaltimer is checked. On expiry the failure code is stored (sys-scope
// release: the word is mapped host memory) and true is returned, so the caller stops waiting.
__device__ __forceinline__ bool spin_expired(const DevStatus& s, unsigned long long t0, uint64_t& spins, uint32_t code) {
  if ((++spins & 1023u) != 0) return false;
  if (gtimer() - t0 < s.timeout_ns) return false;
  if (s.word) asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(s.word), "r"(code) : "memory");
  return true;
}

// Dataflow-mode synchronisation (kFlagDataflow, cgx_args.h).
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// First node, CTA 0, before it triggers: epoch += 1 (the only writer; later nodes read it after
// their launch, which follows this CTA's trigger).
__device__ __forceinline__ void df_bump(const ElemArgs& a) {
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) {
      *a.df_epoch = *a.df_epoch + 1u;
      __threadfence();
    }
    __syncthreads();
  }
}
__device__ __forceinline__ void df_wait(const ElemArgs& a) {
  if (a.df_n == 0) return;
  if (threadIdx.x == 0) {
    const uint32_t ep = ld_relaxed_u32(a.df_epoch);
    for (uint32_t i = 0; i < a.df_n; ++i) {
      const uint32_t target = ep * a.df_ctas[i];
      const uint32_t* c = a.df_done + a.df_dep[i];
      uint64_t spins = 0;
      const unsigned long long t0 = gtimer();
      // poll with relaxed loads (no L1 invalidation per poll), then one acquire fence below; a
      // lost signal is reported through the exec's status word instead of hanging or trapping
      while ((int32_t)(ld_relaxed_u32(c) - target) < 0) {
        if (spin_expired(a.st, t0, spins, kDevErrDataflow)) break;
      }
    }
    asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
  }
  __syncthreads();
}
// bar.sync orders every thread's stores before thread 0's release; a release reduction (cumulative
// over what thread 0 has observed) publishes them together with the count.
__device__ __forceinline__ void df_signal(const ElemArgs& a) {
  __syncthreads();
  if (threadIdx.x == 0)
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" :: "l"(a.df_done + a.df_self) : "memory");
}

// Plain (weak, L1-cached) 16-byte global load through an address that came from the pointer table
// or a by-value param: without the explicit state space the compiler emits a generic LD.
__device__ __forceinline__ float4 ld_global_f4(const float4* p) {
  float4 v;
  asm volatile("ld.global.v4.f32 {%0,%1,%2,%3}, [%4];\n" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p) : "memory");
  return v;
}

// Replay timeline diagnostics (ElemArgs::trace): one thread per CTA stamps %globaltimer.
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// The same replay-timeline stamps for the decoder kernels (one thread per CTA calls it).
// [0] first CTA entry (min), [1] first CTA past its input wait (min), [2] last CTA exit (max): the
// node's work window is [1]..[2] even for grids of several waves (whose last CTAs start late).
// Only the first 256 CTAs stamp entry / ready and only the last 256 stamp the exit: every stamp is
// an atomic on one of three words, and a multi-wave elementwise grid of 16K CTAs serialised ~50K
// same-address atomics (~0.6 ms per replay at the C4 256 MiB point).
__device__ __forceinline__ void node_stamp(unsigned long long* nt, int what) {
  if (nt) {
    const uint32_t cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    const uint32_t ctas = gridDim.x * gridDim.y * gridDim.z;
    if (what < 2 ? cta >= 256u : cta + 256u < ctas) return;
    const unsigned long long t = gtimer();
    if (what < 2) atomicMin(nt + what, t);
    else atomicMax(nt + what, t);
  }
}
__device__ __forceinline__ void trace_at(const ElemArgs& a, int what) {
  if (threadIdx.x == 0) node_stamp(a.trace, what);
}

// Pointer-table entry. Read-only path: the table never changes while a reader kernel runs (it is
// written before the graph starts, by a root node the reader waits for, or by the T5 publisher
// before it triggers the reader's launch), and L1/texture state is invalidated at every kernel
// launch. Through L1 the warps of an SM share one miss instead of each hammering the same L2 line.
__device__ __forceinline__ uint64_t ld_table(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.nc.u64 %0, [%1];\n" : "=l"(v) : "l"(p));
  return v;
}

// Streaming 16-byte load (read-only for the kernel's lifetime, do not allocate in L1).
__device__ __forceinline__ int4 ld_stream16(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream16(void* p, const int4& v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};\n"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

__device__ __forceinline__ uint64_t splitmix_mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace cgx
