// Probe: nested CUDA-graph WHILE conditional nodes built by stream capture, with a
// two-stream fork/join inside the inner body (the pattern Engine G's device-driven
// Algorithm 1 relies on).  Prints the counters and the per-launch time of the graph.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/graph_cond_probe tools/graph_cond_probe.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("ERR %s line %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void inc(int* c, int i) { if (threadIdx.x == 0) atomicAdd(&c[i], 1); }
__global__ void set_inner(cudaGraphConditionalHandle h, int* c) {
  if (threadIdx.x == 0) { c[5]++; cudaGraphSetConditional(h, (c[5] % 4) != 0); }
}
__global__ void set_outer(cudaGraphConditionalHandle h, int* c) {
  if (threadIdx.x == 0) { c[6]++; cudaGraphSetConditional(h, c[6] < 3); }
}
__global__ void empty_exit(const int* flag) { if (*flag) return; }
__global__ void spin(long long cycles) { long long t0 = clock64(); while (clock64() - t0 < cycles) { } }

static int add_while(cudaStream_t st, cudaGraphConditionalHandle* h, cudaGraph_t* body, unsigned init) {
  cudaStreamCaptureStatus cs;
  const cudaGraphNode_t* deps;
  size_t nd;
  cudaGraph_t g;
  CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
  CK(cudaGraphConditionalHandleCreate(h, g, init, cudaGraphCondAssignDefault));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = *h;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, deps, nd, &p));
  *body = p.conditional.phGraph_out[0];
  CK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
  return 0;
}

int main() {
  int* c;
  CK(cudaMalloc(&c, 64));
  CK(cudaMemset(c, 0, 64));
  cudaStream_t s0, s1, s2, s3;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking));
  cudaEvent_t ev1, ev2;
  CK(cudaEventCreateWithFlags(&ev1, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ev2, cudaEventDisableTiming));
  cudaGraph_t top;
  CK(cudaGraphCreate(&top, 0));
  CK(cudaStreamBeginCaptureToGraph(s0, top, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  inc<<<1, 32, 0, s0>>>(c, 0);
  cudaGraphConditionalHandle ho, hi;
  cudaGraph_t bo, bi;
  if (add_while(s0, &ho, &bo, 1)) return 1;
  // outer body
  CK(cudaStreamBeginCaptureToGraph(s1, bo, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  inc<<<1, 32, 0, s1>>>(c, 1);
  if (add_while(s1, &hi, &bi, 1)) return 1;
  {  // inner body: fork to s3 and join
    CK(cudaStreamBeginCaptureToGraph(s2, bi, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    inc<<<1, 32, 0, s2>>>(c, 2);
    CK(cudaEventRecord(ev1, s2));
    CK(cudaStreamWaitEvent(s3, ev1, 0));
    inc<<<1, 32, 0, s3>>>(c, 3);
    CK(cudaEventRecord(ev2, s3));
    inc<<<1, 32, 0, s2>>>(c, 4);
    CK(cudaStreamWaitEvent(s2, ev2, 0));
    set_inner<<<1, 32, 0, s2>>>(hi, c);
    cudaGraph_t tmp;
    CK(cudaStreamEndCapture(s2, &tmp));
  }
  set_outer<<<1, 32, 0, s1>>>(ho, c);
  cudaGraph_t tmp1;
  CK(cudaStreamEndCapture(s1, &tmp1));
  inc<<<1, 32, 0, s0>>>(c, 7);
  cudaGraph_t tmp0;
  CK(cudaStreamEndCapture(s0, &tmp0));
  cudaGraphExec_t ex;
  CK(cudaGraphInstantiate(&ex, top, 0));
  CK(cudaGraphLaunch(ex, s0));
  CK(cudaStreamSynchronize(s0));
  int h[16];
  CK(cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost));
  printf("counters: start %d outer %d inner %d fork %d join %d innerflag %d outerflag %d end %d\n", h[0], h[1], h[2],
         h[3], h[4], h[5], h[6], h[7]);
  printf("expect:   start 1 outer 3 inner 12 fork 12 join 12 innerflag 12 outerflag 3 end 1\n");
  {  // does launching a graph with conditional nodes block the host behind earlier stream work?
    spin<<<1, 1, 0, s0>>>(2000000000LL);
    auto h0 = std::chrono::steady_clock::now();
    CK(cudaGraphLaunch(ex, s0));
    auto h1 = std::chrono::steady_clock::now();
    printf("host time of cudaGraphLaunch behind a ~1 s spin: %.3f ms (query %d)\n",
           std::chrono::duration<double, std::milli>(h1 - h0).count(), (int)cudaStreamQuery(s0));
    CK(cudaStreamSynchronize(s0));
  }
  // timing: empty-exit launches (capture 200 in a graph)
  int* flag;
  CK(cudaMalloc(&flag, 4));
  CK(cudaMemset(flag, 0xff, 4));
  cudaGraph_t g2;
  CK(cudaStreamBeginCapture(s0, cudaStreamCaptureModeRelaxed));
  for (int i = 0; i < 200; ++i) empty_exit<<<dim3(16, 512), 256, 0, s0>>>(flag);
  CK(cudaStreamEndCapture(s0, &g2));
  cudaGraphExec_t ex2;
  CK(cudaGraphInstantiate(&ex2, g2, 0));
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  CK(cudaGraphLaunch(ex2, s0));
  cudaEventRecord(t0, s0);
  CK(cudaGraphLaunch(ex2, s0));
  cudaEventRecord(t1, s0);
  CK(cudaStreamSynchronize(s0));
  float ms;
  cudaEventElapsedTime(&ms, t0, t1);
  printf("empty-exit launch of 16x512 CTAs in a graph: %.2f us each\n", ms * 1000.f / 200);
  cudaGraph_t g3;
  CK(cudaStreamBeginCapture(s0, cudaStreamCaptureModeRelaxed));
  for (int i = 0; i < 200; ++i) empty_exit<<<1, 32, 0, s0>>>(flag);
  CK(cudaStreamEndCapture(s0, &g3));
  cudaGraphExec_t ex3;
  CK(cudaGraphInstantiate(&ex3, g3, 0));
  CK(cudaGraphLaunch(ex3, s0));
  cudaEventRecord(t0, s0);
  CK(cudaGraphLaunch(ex3, s0));
  cudaEventRecord(t1, s0);
  CK(cudaStreamSynchronize(s0));
  cudaEventElapsedTime(&ms, t0, t1);
  printf("1-CTA launch in a graph: %.2f us each\n", ms * 1000.f / 200);
  return 0;
}
