// Microbenchmark (round 2): tcgen05.mma issue and execution rate for the decoder GEMM's tile shape
// (M = 128, N = BN, K = 16 per instruction, bf16 SS operands, SW128 K-major), operands already in
// shared memory (no TMA). One thread issues n_kb k-blocks x 4 MMAs; cycles (clock64) from the first
// issue to the last issue returned, and to the commit barrier firing (execution complete).
// Variants: BN in {32, 64, 128, 256}; per-k-block mbarrier wait on an already-completed barrier
// (the mainloop's per-stage wait) on / off.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_rate_microbench umma_rate_microbench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)(16 >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(tmem), "l"(a), "l"(b), "r"(id), "r"(acc));
}
// whole-warp issue: every lane executes, elect.sync picks one to issue (converged warp)
__device__ __forceinline__ void mma_elect(uint32_t tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p, q;\n elect.sync _|q, 0xffffffff;\n setp.ne.b32 p, %4, 0;\n"
               " @q tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(tmem), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  uint32_t done;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(su32(b)), "r"(ph) : "memory");
  } while (!done);
}

template <int BN, int BM = 128>
__global__ void k_rate(int n_kb, int wait_each, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar_done, bar_ready;
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5;
  uint8_t* sA = smem;                       // [n_kb][128][128 B]
  uint8_t* sB = smem + n_kb * 16384;        // [n_kb][BN][128 B]
  for (int i = threadIdx.x; i < (n_kb * (16384 + BN * 128)) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar_done)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar_ready)));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar_ready)) : "memory");   // phase 0 done
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  constexpr int cols = BN < 32 ? 32 : BN;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s_tmem)), "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  if (threadIdx.x == 32) {
    constexpr uint32_t id = idesc(BM, BN);
    const unsigned long long t0 = clock64();
    for (int kb = 0; kb < n_kb; ++kb) {
      if (wait_each) {
        mb_wait(&bar_ready, 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      const uint64_t da = desc_sw128(su32(sA + kb * 16384)), db = desc_sw128(su32(sB + kb * BN * 128));
#pragma unroll
      for (int k = 0; k < 4; ++k) mma(tmem, da + 2 * k, db + 2 * k, id, (kb | k) != 0);
    }
    const unsigned long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar_done)) : "memory");
    mb_wait(&bar_done, 0);
    const unsigned long long t2 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
  }
}

// n_iss warps (lane 0 each) issue the k-blocks kb = w, w + n_iss, ... into their own accumulator
// (TMEM columns w * BN): intra-CTA split-K, no data exchange.
template <int BN>
__global__ void k_rate_multi(int n_kb, int n_iss, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar_done[4];
  __shared__ uint32_t s_tmem;
  __shared__ unsigned long long t_start;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* sA = smem;
  uint8_t* sB = smem + n_kb * 16384;
  for (int i = threadIdx.x; i < (n_kb * (16384 + BN * 128)) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar_done[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  constexpr int cols = BN * 4 < 32 ? 32 : BN * 4;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s_tmem)), "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  if (threadIdx.x == 0) t_start = clock64();
  __syncthreads();
  if (warp < n_iss && lane == 0) {
    constexpr uint32_t id = idesc(128, BN);
    for (int kb = warp; kb < n_kb; kb += n_iss) {
      const uint64_t da = desc_sw128(su32(sA + kb * 16384)), db = desc_sw128(su32(sB + kb * BN * 128));
#pragma unroll
      for (int k = 0; k < 4; ++k) mma(tmem + warp * BN, da + 2 * k, db + 2 * k, id, (kb != warp) || k);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar_done[warp])) : "memory");
  }
  if (threadIdx.x == 0) {
    for (int w = 0; w < n_iss; ++w) mb_wait(&bar_done[w], 0);
    out[blockIdx.x * 2] = 0;
    out[blockIdx.x * 2 + 1] = clock64() - t_start;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
  }
}

template <int BN>
void run_multi(unsigned long long* d, int n_kb, int n_iss, int clk_khz) {
  const size_t smem = n_kb * (16384 + BN * 128) + 1024;
  if (smem > 220 * 1024) return;
  CK(cudaFuncSetAttribute(k_rate_multi<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  unsigned long long h[2];
  double best = 1e30;
  for (int rep = 0; rep < 5; ++rep) {
    k_rate_multi<BN><<<1, 128, smem>>>(n_kb, n_iss, d);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
    if (h[1] < best) best = (double)h[1];
  }
  printf("MULTI BN %3d kb %2d issuers %d | done %7.0f cyc = %6.3f us (%5.1f cyc/mma overall)\n", BN, n_kb, n_iss, best,
         best / (clk_khz * 1e3) * 1e3, best / (4 * n_kb));
}

template <int BN>
__global__ void k_rate_warp(int n_kb, unsigned long long* out, int n_iss = 1) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar_done, bar_done2;
  __shared__ uint32_t s_tmem;
  __shared__ unsigned long long t_start;
  const int warp = threadIdx.x >> 5;
  uint8_t* sA = smem;
  uint8_t* sB = smem + n_kb * 16384;
  for (int i = threadIdx.x; i < (n_kb * (16384 + BN * 128)) / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0, 0);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar_done)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar_done2)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  constexpr int cols = BN < 32 ? 64 : 2 * BN;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&s_tmem)), "r"(cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  if (threadIdx.x == 0) t_start = clock64();
  __syncthreads();
  if (warp >= 1 && warp <= n_iss) {
    const int w = warp - 1;
    constexpr uint32_t id = idesc(128, BN);
    const unsigned long long t0 = t_start;
    for (int kb = w; kb < n_kb; kb += n_iss) {
      const uint64_t da = desc_sw128(su32(sA + kb * 16384)), db = desc_sw128(su32(sB + kb * BN * 128));
#pragma unroll
      for (int k = 0; k < 4; ++k) mma_elect(tmem + w * BN, da + 2 * k, db + 2 * k, id, (kb != w) || k);
    }
    const unsigned long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) {
      uint64_t* b = w == 0 ? &bar_done : &bar_done2;
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(b)) : "memory");
      mb_wait(b, 0);
      if (w == 0) {
        if (n_iss == 2) mb_wait(&bar_done2, 0);
        out[0] = t1 - t0;
        out[1] = clock64() - t0;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(cols));
  }
}
template <int BN>
void run_warp(unsigned long long* d, int n_kb, int n_iss = 1) {
  const size_t smem = n_kb * (16384 + BN * 128) + 1024;
  CK(cudaFuncSetAttribute(k_rate_warp<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  unsigned long long h[2];
  double bi = 1e30, be = 1e30;
  for (int rep = 0; rep < 5; ++rep) {
    k_rate_warp<BN><<<1, 128, smem>>>(n_kb, d, n_iss);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
    if (h[0] < bi) bi = (double)h[0];
    if (h[1] < be) be = (double)h[1];
  }
  printf("WARP x%d ", n_iss);
  printf("BN %3d kb %2d | issue %6.0f cyc (%5.1f /mma) | done %6.0f cyc (%5.1f /mma)\n", BN, n_kb, bi, bi / (4 * n_kb), be,
         be / (4 * n_kb));
}

template <int BN, int BM = 128>
void run(unsigned long long* d, int n_kb, int wait_each, int ctas, int clk_khz) {
  const size_t smem = n_kb * (16384 + BN * 128) + 1024;
  if (smem > 220 * 1024) return;
  CK(cudaFuncSetAttribute(k_rate<BN, BM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  unsigned long long h[2 * 148];
  double best_i = 1e30, best_e = 1e30;
  for (int rep = 0; rep < 5; ++rep) {
    k_rate<BN, BM><<<ctas, 128, smem>>>(n_kb, wait_each, d);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h, d, sizeof(unsigned long long) * 2 * ctas, cudaMemcpyDeviceToHost));
    if (h[0] < best_i) best_i = (double)h[0];
    if (h[1] < best_e) best_e = (double)h[1];
  }
  const double flop = 2.0 * BM * BN * 64 * n_kb;
  printf("BM %3d ", BM);
  printf("BN %3d kb %2d wait %d ctas %3d | issue %7.0f cyc (%5.1f cyc/mma) | done %7.0f cyc (%5.1f cyc/mma, %6.2f ns/kb) | %.2f TFLOP/s/SM @%.2f GHz\n",
         BN, n_kb, wait_each, ctas, best_i, best_i / (4 * n_kb), best_e, best_e / (4 * n_kb),
         best_e / (4 * n_kb) * 4 / (clk_khz * 1e-6), flop / (best_e / (clk_khz * 1e3)) / 1e12, clk_khz * 1e-6);
}

int main() {
  unsigned long long* d;
  CK(cudaMalloc(&d, sizeof(unsigned long long) * 2 * 148));
  int clk = 0;
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  for (int kb : {4, 8}) {
    for (int iss : {1, 2}) {
      run_warp<32>(d, kb, iss);
      run_warp<64>(d, kb, iss);
    }
  }
  return 0;
  for (int kb : {4, 8}) {
    run<32, 64>(d, kb, 0, 1, clk);
    run<64, 64>(d, kb, 0, 1, clk);
    run<128, 64>(d, kb, 0, 1, clk);
    run<32, 64>(d, kb, 1, 1, clk);
    run<32, 128>(d, kb, 0, 1, clk);
  }
  for (int w : {0, 1})
    for (int kb : {1, 4, 12}) {
      run<32>(d, kb, w, 1, clk);
      run<64>(d, kb, w, 1, clk);
      run<128>(d, kb, w, 1, clk);
      run<256>(d, kb, w, 1, clk);
    }
  for (int iss : {1, 2, 3, 4}) {
    run_multi<32>(d, 8, iss, clk);
    run_multi<32>(d, 10, iss, clk);
    run_multi<16>(d, 12, iss, clk);
  }
  return 0;
}
