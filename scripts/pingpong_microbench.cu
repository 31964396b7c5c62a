// Inter-SM flag round trip on B200: CTA 0 and CTA 1 (on different SMs) bounce a counter through
// global memory n times; one-way latency = span / (2 n). Variants of the store / poll instructions.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/pingpong_microbench scripts/pingpong_microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int V>
__device__ __forceinline__ void st(uint32_t* p, uint32_t v) {
  if (V == 0) asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  if (V == 1) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  if (V == 2) asm volatile("st.volatile.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  if (V == 3) asm volatile("atom.exch.relaxed.gpu.global.b32 _, [%0], %1;" ::"l"(p), "r"(v) : "memory");
  if (V == 4) asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <int V>
__device__ __forceinline__ uint32_t ld(const uint32_t* p) {
  uint32_t v;
  if (V == 0) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  if (V == 1) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  if (V == 2) asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  if (V == 3) asm volatile("atom.add.relaxed.gpu.global.u32 %0, [%1], 0;" : "=r"(v) : "l"(p) : "memory");
  if (V == 4) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int S, int L>
__global__ void pingpong(uint32_t* f, int n, unsigned long long* out) {
  if (threadIdx.x != 0) return;
  uint32_t* a = f;            // written by CTA 0
  uint32_t* b = f + 64;       // written by CTA 1 (other line)
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 1; i <= n; ++i) {
    if (blockIdx.x == 0) {
      st<S>(a, i);
      while (ld<L>(b) != (uint32_t)i) {}
    } else if (blockIdx.x == gridDim.x - 1) {
      while (ld<L>(a) != (uint32_t)i) {}
      st<S>(b, i);
    }
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (blockIdx.x == 0) out[0] = t1 - t0;
}

template <int S, int L>
void run(const char* name, uint32_t* f, unsigned long long* d_out, int ctas) {
  const int n = 20000;
  cudaMemset(f, 0, 4096);
  pingpong<S, L><<<ctas, 32>>>(f, n, d_out);
  cudaDeviceSynchronize();
  cudaMemset(f, 0, 4096);
  pingpong<S, L><<<ctas, 32>>>(f, n, d_out);
  unsigned long long ns = 0;
  cudaMemcpy(&ns, d_out, 8, cudaMemcpyDeviceToHost);
  printf("%-36s ctas %3d one-way %7.1f ns\n", name, ctas, ns / (2.0 * n));
}

int main() {
  uint32_t* f;
  unsigned long long* d_out;
  cudaMalloc(&f, 4096);
  cudaMalloc(&d_out, 8);
  for (int ctas : {2, 148}) {
    run<0, 0>("st.relaxed.gpu / ld.relaxed.gpu", f, d_out, ctas);
    run<1, 1>("st.release.gpu / ld.acquire.gpu", f, d_out, ctas);
    run<2, 2>("st.volatile / ld.volatile", f, d_out, ctas);
    run<3, 3>("atom.exch / atom.add 0", f, d_out, ctas);
    run<4, 0>("red.max / ld.relaxed.gpu", f, d_out, ctas);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
