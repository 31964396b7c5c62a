// Stand-alone microbenchmark: the PDL launch cadence of a captured chain of short kernels on
// sm_100a. A graph of K kernels, each triggering its dependent at entry (griddepcontrol.
// launch_dependents) and optionally waiting (griddepcontrol.wait), replayed back to back; reports
// µs per kernel for varying parameter size, CTA size, grid size and per-thread work.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_microbench launch_microbench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int PB>
struct P { float* out; uint32_t n; uint32_t wait; uint8_t pad[PB]; };

template <int PB, int V = 0>
__global__ void k_chain(const __grid_constant__ P<PB> p) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (p.wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < p.n) p.out[i] = p.out[i] * (0.5f + V) + 1.0f;
}

// In-flight depth of the PDL cascade: each kernel triggers at entry, then busy-waits `ns`.
__global__ void k_sleep(unsigned long long ns) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < ns);
}

static double run_sleep(int K, int grid, unsigned long long ns, int reps) {
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int k = 0; k < K; ++k) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(32);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k_sleep, ns));
  }
  CK(cudaStreamEndCapture(s, &g));
  cudaGraphExec_t ge;
  CK(cudaGraphInstantiate(&ge, g, 0));
  for (int i = 0; i < 5; ++i) CK(cudaGraphLaunch(ge, s));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaStreamSynchronize(s));
  CK(cudaEventRecord(e0, s));
  for (int i = 0; i < reps; ++i) CK(cudaGraphLaunch(ge, s));
  CK(cudaEventRecord(e1, s));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
  return ms * 1e3 / reps / K;
}

// nfn distinct kernel functions used round-robin (instruction-cache / function-switch cost)
template <int PB>
static double run(int K, int grid, int block, int wait, int reps, float* buf, int nfn = 1) {
  cudaStream_t s;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaGraph_t g;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
  for (int k = 0; k < K; ++k) {
    P<PB> p{};
    p.out = buf;
    p.n = (uint32_t)grid * block;
    p.wait = wait;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const int f = k % nfn;
    if (f == 0) CK(cudaLaunchKernelEx(&cfg, k_chain<PB, 0>, p));
    else if (f == 1) CK(cudaLaunchKernelEx(&cfg, k_chain<PB, 1>, p));
    else CK(cudaLaunchKernelEx(&cfg, k_chain<PB, 2>, p));
  }
  CK(cudaStreamEndCapture(s, &g));
  cudaGraphExec_t ge;
  CK(cudaGraphInstantiate(&ge, g, 0));
  for (int i = 0; i < 20; ++i) CK(cudaGraphLaunch(ge, s));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaStreamSynchronize(s));
  CK(cudaEventRecord(e0, s));
  for (int i = 0; i < reps; ++i) CK(cudaGraphLaunch(ge, s));
  CK(cudaEventRecord(e1, s));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
  return ms * 1e3 / reps / K;
}

int main() {
  float* buf;
  CK(cudaMalloc(&buf, 64 << 20));
  CK(cudaMemset(buf, 0, 64 << 20));
  const int K = 200, reps = 200;
  printf("K=%d kernels per graph, us per kernel\n", K);
  printf("PDL cascade depth: kernels trigger at entry then run for T us (no wait)\n%6s %8s %8s %10s\n", "grid", "T_us", "us/kern", "T/us_kern");
  for (int grid : {1, 16})
    for (unsigned long long ns : {0ull, 500ull, 1000ull, 2000ull, 4000ull, 8000ull, 16000ull}) {
      const double u = run_sleep(K, grid, ns, 50);
      printf("%6d %8.1f %8.3f %10.2f\n", grid, ns / 1e3, u, ns / 1e3 / u);
    }
  printf("function switching (params 160 B, block 256):\n%6s %5s %8s %8s\n", "grid", "wait", "1 fn", "3 fns");
  for (int wait = 0; wait <= 1; ++wait)
    for (int grid : {1, 16, 256})
      printf("%6d %5d %8.3f %8.3f\n", grid, wait, run<144>(K, grid, 256, wait, reps, buf, 1),
             run<144>(K, grid, 256, wait, reps, buf, 3));
  printf("%-10s %6s %6s %5s %8s\n", "params_B", "grid", "block", "wait", "us/kern");
  for (int wait = 0; wait <= 1; ++wait)
    for (int block : {32, 256})
      for (int grid : {1, 16, 148, 512, 1184}) {
        printf("%-10d %6d %6d %5d %8.3f\n", 16, grid, block, wait, run<8>(K, grid, block, wait, reps, buf));
        printf("%-10d %6d %6d %5d %8.3f\n", 160, grid, block, wait, run<144>(K, grid, block, wait, reps, buf));
        printf("%-10d %6d %6d %5d %8.3f\n", 4096, grid, block, wait, run<4080>(K, grid, block, wait, reps, buf));
      }
  return 0;
}
