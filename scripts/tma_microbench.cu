// Stand-alone microbenchmark: per-SM TMA ingress from L2. The C3 decoder GEMM (k_gemm_bf16, M = 128)
// spends ~0.3 us per 20 KB k-block stage at 24, 72 or 96 CTAs alike (profiles/r01/
// gemm_tiling_trace_sweep.txt), i.e. ~34 B/clk per SM, independent of how many SMs run — so the
// question is what one SM's TMA path sustains from an L2-resident operand, and whether ring depth,
// box size or sharing the same lines across CTAs (the activation tile every N-tile reads) moves it.
//
// Kernel: one producer thread streams `iters` 2-D boxes (rows x bw bf16, no swizzle) of an L2-resident bf16 tensor [128][cols] into a ring of `stages` slots; one consumer
// thread waits each slot's full barrier and releases it at once (no compute). Per CTA the
// globaltimer span from the first issue to the last arrival gives bytes/ns; reported: median over
// CTAs, in GB/s per SM and B/clk at the measured SM clock.
//   same=1: every CTA reads the same column range (the GEMM's shared A operand)
//   same=0: CTA b reads its own columns (distinct lines)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_microbench tma_microbench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

static __device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
static __device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
static __device__ __forceinline__ void mb_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
static __device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
static __device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
static __device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  uint32_t done;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(su32(b)), "r"(ph) : "memory");
  } while (!done);
}
static __device__ __forceinline__ void mb_spin(uint64_t* b, uint32_t ph) {   // test_wait: never suspends
  uint32_t done;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(su32(b)), "r"(ph) : "memory");
  } while (!done);
}
static __device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* tm, uint64_t* bar, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(su32(dst)), "l"(tm), "r"(su32(bar)), "r"(x), "r"(y) : "memory");
}

__global__ void k_ingress(const __grid_constant__ CUtensorMap tm, int rows, int bw, int stages, int iters, int same,
                          int cols_per_cta, int flags, uint64_t* span_ns) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t box = (uint32_t)rows * (uint32_t)bw * 2u;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * box);
  uint64_t* empty = full + stages;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int c0 = same ? 0 : (blockIdx.x % 148) * cols_per_cta;
  const int nblk = cols_per_cta / bw;
  __shared__ uint64_t t0;
  // flags & 4: two producer warps (warp 0 issues even boxes, warp 2 odd ones)
  const int nprod = (flags & 4) ? 2 : 1;
  const int prod = threadIdx.x == 0 ? 0 : (nprod == 2 && threadIdx.x == 64) ? 1 : -1;
  if (threadIdx.x == 0) t0 = gtime();
  if (prod >= 0) {
    if (flags & 1) asm volatile("prefetch.tensormap [%0];" ::"l"(&tm) : "memory");
    for (int i = prod; i < iters; i += nprod) {
      const int s = i % stages;
      if (i >= stages) {
        if (flags & 2) mb_spin(&empty[s], (uint32_t)((i / stages) - 1) & 1u);
        else mb_wait(&empty[s], (uint32_t)((i / stages) - 1) & 1u);
      }
      mb_expect(&full[s], box);
      tma2d(smem + (size_t)s * box, &tm, &full[s], c0 + (i % nblk) * bw, 0);
    }
  } else if (threadIdx.x == 32) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % stages;
      if (flags & 2) mb_spin(&full[s], (uint32_t)(i / stages) & 1u);
      else mb_wait(&full[s], (uint32_t)(i / stages) & 1u);
      mb_arrive(&empty[s]);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) span_ns[blockIdx.x] = gtime() - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeFn encode = reinterpret_cast<EncodeFn>(fn);
  const int R = 128;
  const int COLS = 65536;   // [128][65536] bf16 = 16 MiB: L2-resident
  void* buf;
  CK(cudaMalloc(&buf, (size_t)R * COLS * 2));
  CK(cudaMemset(buf, 0, (size_t)R * COLS * 2));
  uint64_t* d_span;
  CK(cudaMalloc(&d_span, 296 * sizeof(uint64_t)));
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  CK(cudaFuncSetAttribute(k_ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  printf("per-SM TMA ingress from L2 (box rows x bw bf16, no swizzle, ring of `stages`); GB/s per SM = median over CTAs\n");
  printf("flags: 1 = prefetch.tensormap, 2 = test_wait spin instead of try_wait, 4 = two producer warps; 296 ctas = 2 per SM\n");
  printf("%5s %5s %5s %8s %7s %5s %5s %10s %10s %10s %9s\n", "flags", "rows", "bw", "box_KB", "stages", "ctas", "same", "GB/s/SM",
         "B/clk", "chip_GB/s", "ns/box");
  struct Cfg { int rows, bw, stages; };
  const Cfg cfgs[] = {{8, 64, 8}, {32, 64, 8}, {32, 64, 40}, {64, 64, 8}, {128, 64, 4}, {128, 64, 8}, {256, 64, 4},
                      {128, 128, 4}, {128, 256, 3}, {256, 128, 3}, {256, 256, 1}, {32, 256, 8}, {128, 64, 12}};
  const int only_flags = argc > 1 ? atoi(argv[1]) : -1;
  for (int flags : {0, 4, 6})
  for (const Cfg& c : cfgs)
    for (int ctas : {1, 148, 296})
      for (int same : {1, 0}) {
        if (only_flags >= 0 && flags != only_flags) continue;
        if (ctas == 296 && (c.stages * c.rows * c.bw * 2 > 100 * 1024)) continue;
        const int rows = c.rows, bw = c.bw, stages = c.stages;
        const uint32_t box = (uint32_t)rows * (uint32_t)bw * 2u;
        if ((size_t)stages * box + 1024 > 220 * 1024) continue;
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)COLS, (cuuint64_t)R};
        cuuint64_t strides[1] = {(cuuint64_t)COLS * 2};
        cuuint32_t boxd[2] = {(cuuint32_t)bw, (cuuint32_t)rows};
        cuuint32_t es[2] = {1, 1};
        if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, boxd, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
          printf("encode failed rows=%d bw=%d\n", rows, bw);
          continue;
        }
        const int cols_per_cta = 256 * 1;   // window per CTA (same=0): distinct lines per CTA (wraps at 296)
        const int iters = 96;
        const size_t smem = (size_t)stages * box + 2 * stages * sizeof(uint64_t) + 64;
        std::vector<double> gbs;
        for (int rep = 0; rep < 6; ++rep) {
          k_ingress<<<ctas, 96, smem>>>(tm, rows, bw, stages, iters, same, cols_per_cta, flags, d_span);
          CK(cudaGetLastError());
          CK(cudaDeviceSynchronize());
          if (rep < 2) continue;   // warm L2
          std::vector<uint64_t> sp(ctas);
          CK(cudaMemcpy(sp.data(), d_span, ctas * sizeof(uint64_t), cudaMemcpyDeviceToHost));
          std::sort(sp.begin(), sp.end());
          gbs.push_back((double)iters * box / (double)sp[ctas / 2]);
        }
        std::sort(gbs.begin(), gbs.end());
        const double g = gbs[gbs.size() / 2];
        printf("%5d %5d %5d %8.1f %7d %5d %5d %10.1f %10.1f %10.0f %9.1f\n", flags, rows, bw, box / 1024.0, stages, ctas, same, g,
               g / (clk_khz * 1e-6), g * ctas, box / g);
      }
  return 0;
}
