// Stand-alone microbenchmark of multi-tensor copy kernel variants on sm_100a (3 x 1 GiB).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o copy_microbench copy_microbench.cu
// Every variant is timed in 4 interleaved rounds (10 launches each, median), to average out the
// run-to-run HBM noise seen on this pool.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <functional>
#include <string>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

struct Args { const int4* src[3]; int4* dst[3]; uint64_t n16[3]; };

__device__ __forceinline__ int4 ldnc(const int4* p) {
  int4 r; asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p)); return r;
}
__device__ __forceinline__ void stna(int4* p, int4 v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// grid-stride per tensor, U loads in flight per thread
template <int U, bool NC>
__global__ void k_gs(const __grid_constant__ Args a) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (int t = 0; t < 3; ++t) {
    const int4* s = a.src[t]; int4* d = a.dst[t]; const uint64_t n = a.n16[t];
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n; i += U * stride) {
      int4 v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) v[j] = NC ? ldnc(s + i + j * stride) : s[i + j * stride];
#pragma unroll
      for (int j = 0; j < U; ++j) { if (NC) stna(d + i + j * stride, v[j]); else d[i + j * stride] = v[j]; }
    }
    for (; i < n; i += stride) d[i] = s[i];
  }
}

// grid-stride where each thread handles U CONSECUTIVE vectors of a warp-contiguous block
template <int U>
__global__ void k_gsw(const __grid_constant__ Args a) {
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = nthreads >> 5;
  for (int t = 0; t < 3; ++t) {
    const int4* s = a.src[t]; int4* d = a.dst[t]; const uint64_t n = a.n16[t];
    for (uint64_t b = warp * (32 * U); b < n; b += nwarps * (32 * U)) {
      int4 v[U];
#pragma unroll
      for (int j = 0; j < U; ++j) { const uint64_t i = b + j * 32 + lane; if (i < n) v[j] = s[i]; }
#pragma unroll
      for (int j = 0; j < U; ++j) { const uint64_t i = b + j * 32 + lane; if (i < n) d[i] = v[j]; }
    }
  }
}

int main() {
  const uint64_t S = 1ull << 30;
  Args a;
  for (int t = 0; t < 3; ++t) {
    void *s, *d;
    CK(cudaMalloc(&s, S)); CK(cudaMalloc(&d, S));
    CK(cudaMemset(s, t + 1, S)); CK(cudaMemset(d, 0, S));
    a.src[t] = (const int4*)s; a.dst[t] = (int4*)d; a.n16[t] = S / 16;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  struct V { std::string name; std::function<void()> f; std::vector<double> med; };
  std::vector<V> vs;
  vs.push_back({"memcpyAsync x3", [&] { for (int t = 0; t < 3; ++t) cudaMemcpyAsync(a.dst[t], a.src[t], S, cudaMemcpyDeviceToDevice); }, {}});
  for (int blk : {256, 512, 1024})
    for (int cps : {1, 2, 4, 8}) {
      const int g = 148 * cps;
      if (blk * cps > 2048) continue;
      char nm[96];
      snprintf(nm, 96, "gs U1 plain b=%d g=%d", blk, g); vs.push_back({nm, [=, &a] { k_gs<1, false><<<g, blk>>>(a); }, {}});
      snprintf(nm, 96, "gs U2 plain b=%d g=%d", blk, g); vs.push_back({nm, [=, &a] { k_gs<2, false><<<g, blk>>>(a); }, {}});
      snprintf(nm, 96, "gs U4 plain b=%d g=%d", blk, g); vs.push_back({nm, [=, &a] { k_gs<4, false><<<g, blk>>>(a); }, {}});
      snprintf(nm, 96, "gs U2 nc b=%d g=%d", blk, g); vs.push_back({nm, [=, &a] { k_gs<2, true><<<g, blk>>>(a); }, {}});
      snprintf(nm, 96, "gsw U4 b=%d g=%d", blk, g); vs.push_back({nm, [=, &a] { k_gsw<4><<<g, blk>>>(a); }, {}});
      snprintf(nm, 96, "gsw U8 b=%d g=%d", blk, g); vs.push_back({nm, [=, &a] { k_gsw<8><<<g, blk>>>(a); }, {}});
    }
  for (int round = 0; round < 4; ++round)
    for (auto& v : vs) {
      std::vector<float> t;
      for (int r = 0; r < 12; ++r) {
        cudaEventRecord(e0); v.f(); cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (r >= 2) t.push_back(ms);
      }
      std::sort(t.begin(), t.end());
      v.med.push_back(t[t.size() / 2]);
    }
  std::sort(vs.begin(), vs.end(), [](const V& x, const V& y) {
    auto m = [](std::vector<double> q) { std::sort(q.begin(), q.end()); return (q[1] + q[2]) / 2; };
    return m(x.med) < m(y.med);
  });
  for (auto& v : vs) {
    std::vector<double> q = v.med; std::sort(q.begin(), q.end());
    const double ms = (q[1] + q[2]) / 2;
    printf("%-32s %8.1f us  %7.1f GB/s   (rounds:", v.name.c_str(), ms * 1e3, 6.0 * S / (ms * 1e-3) / 1e9);
    for (double x : v.med) printf(" %.0f", 6.0 * S / (x * 1e-3) / 1e9);
    printf(")\n");
  }
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
  return 0;
}
