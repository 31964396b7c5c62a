// Stand-alone microbenchmark: does a captured graph with independent BRANCHES launch its kernels
// faster than one serial PDL chain of the same kernels? C2 is 64 independent lanes of
// ADD -> MUL -> REDUCE; its serial single-stream capture is bound by the PDL launch cadence
// (~0.55-0.6 us per kernel, launch_microbench.cu). Here: B branches x L kernels each, captured
// from B streams (fork/join with events), PDL inside each branch (every kernel triggers at entry and
// griddepcontrol.wait's for its branch predecessor), versus the same B*L kernels on one stream.
// Each kernel: G CTAs x 256 threads, one 16-B load + store per thread (a memory-touching node).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dag_microbench dag_microbench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k_node(float4* buf, uint32_t n4, int wait) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (wait) asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n4) {
    float4 v = buf[i];
    v.x += 1.f;
    buf[i] = v;
  }
}

static void launch(cudaStream_t s, float4* p, uint32_t grid, int wait, bool pdl) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  if (pdl) {
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
  }
  CK(cudaLaunchKernelEx(&cfg, k_node, p, grid * 256u, wait));
}

// B branches x L kernels; nstreams capture streams (branches round-robin); 1 stream = serial chain
// nstreams == 0: one stream, kernels never wait (the dataflow replay's launch-order lower bound)
static double run(int B, int L, uint32_t grid, int nstreams, bool pdl, float4* buf, int reps) {
  const int nowait = nstreams == 0;
  if (nowait) nstreams = 1;
  cudaStream_t origin;
  CK(cudaStreamCreateWithFlags(&origin, cudaStreamNonBlocking));
  std::vector<cudaStream_t> ss(nstreams);
  for (auto& s : ss) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaEvent_t fork;
  CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  std::vector<cudaEvent_t> joins(nstreams);
  for (auto& ev : joins) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CK(cudaStreamBeginCapture(origin, cudaStreamCaptureModeGlobal));
  CK(cudaEventRecord(fork, origin));
  for (auto& s : ss) CK(cudaStreamWaitEvent(s, fork, 0));
  const size_t per = (size_t)grid * 256;
  if (nstreams == 1) {
    // serial order of a single-stream program: lane-major (ADD, MUL, REDUCE of lane 0, then lane 1...)
    for (int b = 0; b < B; ++b)
      for (int l = 0; l < L; ++l) launch(ss[0], buf + (size_t)b * per, grid, nowait ? 0 : 1, pdl);
  } else {
    for (int b = 0; b < B; ++b)
      for (int l = 0; l < L; ++l) launch(ss[b % nstreams], buf + (size_t)b * per, grid, 1, pdl);
  }
  for (int i = 0; i < nstreams; ++i) {
    CK(cudaEventRecord(joins[i], ss[i]));
    CK(cudaStreamWaitEvent(origin, joins[i], 0));
  }
  cudaGraph_t g;
  CK(cudaStreamEndCapture(origin, &g));
  cudaGraphExec_t ge;
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphUpload(ge, origin));
  for (int i = 0; i < 20; ++i) CK(cudaGraphLaunch(ge, origin));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaStreamSynchronize(origin));
  CK(cudaEventRecord(e0, origin));
  for (int i = 0; i < reps; ++i) CK(cudaGraphLaunch(ge, origin));
  CK(cudaEventRecord(e1, origin));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  for (auto& s : ss) cudaStreamDestroy(s);
  cudaStreamDestroy(origin);
  return ms * 1e3 / reps;
}

int main() {
  float4* buf;
  CK(cudaMalloc(&buf, 512 << 20));
  CK(cudaMemset(buf, 0, 512 << 20));
  printf("B branches x L kernels (G CTAs x 256 thr each), us per graph replay\n");
  printf("%4s %3s %5s %9s %9s %9s %9s %9s %9s\n", "B", "L", "G", "ser_nowt", "serial", "2 str", "4 str", "8 str", "B str");
  for (uint32_t G : {1u, 16u, 148u})
    for (int B : {8, 64}) {
      const int L = 3;
      const double s0 = run(B, L, G, 0, true, buf, 100);
      const double s1 = run(B, L, G, 1, true, buf, 100);
      const double s2 = run(B, L, G, 2, true, buf, 100);
      const double s4 = run(B, L, G, 4, true, buf, 100);
      const double s8 = run(B, L, G, 8, true, buf, 100);
      const double sb = run(B, L, G, B, true, buf, 100);
      printf("%4d %3d %5u %9.1f %9.1f %9.1f %9.1f %9.1f %9.1f\n", B, L, G, s0, s1, s2, s4, s8, sb);
    }
  printf("same, without PDL (plain graph edges):\n");
  for (uint32_t G : {1u, 148u}) {
    const int B = 64, L = 3;
    printf("%4d %3d %5u %9.1f %9.1f %9.1f %9.1f %9.1f\n", B, L, G, run(B, L, G, 1, false, buf, 100),
           run(B, L, G, 2, false, buf, 100), run(B, L, G, 4, false, buf, 100), run(B, L, G, 8, false, buf, 100),
           run(B, L, G, B, false, buf, 100));
  }
  return 0;
}
