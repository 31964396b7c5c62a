// Microbenchmark (round 2): how fast can ONE SM pull a GEMM operand slice (A panel [128][K] bf16,
// K-major, SWIZZLE_128B as the decoder GEMM uses) from L2 with TMA, depending on HOW the boxes are
// issued. Each CTA loads `kb` k-blocks (16 KiB each) of the same L2-resident [128][3072] bf16 tensor:
//   mode 0: 2-D boxes {64, 128} (one k-block each), issued by `P` producers
//   mode 1: 3-D boxes {64, 128, G} over the {64, rows, K/64} view (G k-blocks per box), `P` producers
// producers: lanes 0..P-1 of warp 0 (layout 0) or lane 0 of warps 0..P-1 (layout 1).
// All boxes complete on one mbarrier (expect_tx of the total); span = %globaltimer from before
// the first issue to the barrier completion, per CTA; median over CTAs, 1 and 144 CTAs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_issue_microbench tma_issue_microbench.cu
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

__global__ void k_load(const __grid_constant__ CUtensorMap tm2, const __grid_constant__ CUtensorMap tm3, int mode, int kb,
                       int G, int P, int layout, uint64_t* span_ns) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint64_t t0;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm2) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm3) : "memory");
  }
  __syncthreads();
  if (tid == 0) {
    t0 = gtime();
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(kb * 16384) : "memory");
  }
  __syncthreads();
  const int me = layout == 0 ? (warp == 0 && lane < P ? lane : -1) : (lane == 0 && warp < P ? warp : -1);
  if (me >= 0) {
    if (mode == 0) {
      for (int i = me; i < kb; i += P)
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
                     ::"r"(su32(smem + (size_t)i * 16384)), "l"(&tm2), "r"(su32(&bar)), "r"(i * 64), "r"(0) : "memory");
    } else {
      const int nb = (kb + G - 1) / G;
      for (int b = me; b < nb; b += P)
        asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                     ::"r"(su32(smem + (size_t)b * G * 16384)), "l"(&tm3), "r"(su32(&bar)), "r"(0), "r"(0), "r"(b * G) : "memory");
    }
  }
  if (tid == 0) {
    uint32_t done;
    do {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(su32(&bar)), "r"(0) : "memory");
    } while (!done);
    span_ns[blockIdx.x] = gtime() - t0;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeFn encode = reinterpret_cast<EncodeFn>(fn);
  const int M = 128, K = 3072;
  void* buf;
  CK(cudaMalloc(&buf, (size_t)M * K * 2));
  CK(cudaMemset(buf, 0, (size_t)M * K * 2));
  uint64_t* d_span;
  CK(cudaMalloc(&d_span, 148 * sizeof(uint64_t)));
  CK(cudaFuncSetAttribute(k_load, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CUtensorMap tm2, tm3[9];
  {
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M};
    cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    if (encode(&tm2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
      printf("encode2 failed\n");
  }
  for (int G = 1; G <= 8; ++G) {
    cuuint64_t dims[3] = {64, (cuuint64_t)M, (cuuint64_t)K / 64};
    cuuint64_t strides[2] = {(cuuint64_t)K * 2, 128};
    cuuint32_t box[3] = {64, 128, (cuuint32_t)G};
    cuuint32_t es[3] = {1, 1, 1};
    if (encode(&tm3[G], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE))
      printf("encode3 G=%d failed\n", G);
  }
  printf("%4s %3s %3s %3s %6s %5s %9s %9s %9s\n", "mode", "kb", "G", "P", "layout", "ctas", "span_us", "GB/s/SM", "ns/box");
  struct Cfg { int mode, kb, G, P, layout; };
  std::vector<Cfg> cfgs;
  for (int kb : {6, 12}) {
    for (int P : {1, 2, 4, 6, 12}) for (int layout : {0, 1}) if (!(layout == 1 && P > 6)) cfgs.push_back({0, kb, 1, P, layout});
    for (int G : {2, 3, 6}) for (int P : {1, 2, 3}) cfgs.push_back({1, kb, G, P, 1});
  }
  for (const Cfg& c : cfgs)
    for (int ctas : {1, 144}) {
      std::vector<double> sp_us;
      for (int rep = 0; rep < 7; ++rep) {
        k_load<<<ctas, 192, c.kb * 16384 + 2048>>>(tm2, tm3[c.G], c.mode, c.kb, c.G, c.P, c.layout, d_span);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        if (rep < 2) continue;
        std::vector<uint64_t> sp(ctas);
        CK(cudaMemcpy(sp.data(), d_span, ctas * sizeof(uint64_t), cudaMemcpyDeviceToHost));
        std::sort(sp.begin(), sp.end());
        sp_us.push_back(sp[ctas / 2] / 1e3);
      }
      std::sort(sp_us.begin(), sp_us.end());
      const double s = sp_us[sp_us.size() / 2];
      const int nbox = c.mode == 0 ? c.kb : (c.kb + c.G - 1) / c.G;
      printf("%4d %3d %3d %3d %6d %5d %9.3f %9.1f %9.1f\n", c.mode, c.kb, c.G, c.P, c.layout, ctas, s,
             c.kb * 16384 / (s * 1e3), s * 1e3 / nbox);
    }
  return 0;
}
