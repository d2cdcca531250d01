// launch_ub.cu — launch-path costs on this box (diagnostic): plain launch,
// with the runtime calls of the drop-in path around it, a CUDA graph launch,
// and a graph launch with in-place kernel-parameter update.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -cudart static -o tools/launch_ub tools/launch_ub.cu
#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
struct Big { const double* a; const unsigned long long* b; size_t n, ld; unsigned long long s; double dt; void* o; void* f; unsigned* c; double* fs; volatile unsigned* ff; unsigned long long* ops; };
__global__ void k_big(Big b) { if (b.n == 12345) printf("x"); }
int main() {
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  Big b{};
  auto t = [&](const char* name, auto fn) {
    for (int i = 0; i < 50; ++i) { fn(); cudaStreamSynchronize(st); }
    double acc = 0, accrt = 0;
    for (int i = 0; i < 200; ++i) {
      auto a0 = std::chrono::steady_clock::now();
      fn();
      auto a1 = std::chrono::steady_clock::now();
      cudaStreamSynchronize(st);
      auto a2 = std::chrono::steady_clock::now();
      acc += std::chrono::duration<double, std::micro>(a1 - a0).count();
      accrt += std::chrono::duration<double, std::micro>(a2 - a0).count();
    }
    printf("%-40s launch %.2f us, launch+sync %.2f us\n", name, acc / 200, accrt / 200);
  };
  t("plain <<<512,32>>>", [&] { k_big<<<512, 32, 0, st>>>(b); });
  t("setdevice + launch + getlasterror", [&] { cudaSetDevice(0); k_big<<<512, 32, 0, st>>>(b); cudaGetLastError(); });
  cudaPointerAttributes at; void* hp; cudaHostAlloc(&hp, 1 << 20, cudaHostAllocMapped);
  t("2x ptrattr + launch", [&] { cudaPointerGetAttributes(&at, hp); cudaPointerGetAttributes(&at, hp); k_big<<<512, 32, 0, st>>>(b); });
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal); k_big<<<512, 32, 0, st>>>(b); cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  t("graph launch", [&] { cudaGraphLaunch(ge, st); });
  size_t nn = 0; cudaGraphGetNodes(g, nullptr, &nn); cudaGraphNode_t node; nn = 1; cudaGraphGetNodes(g, &node, &nn);
  cudaKernelNodeParams kp; cudaGraphKernelNodeGetParams(node, &kp);
  Big b2{}; void* args[1] = {&b2};
  t("setparams + graph launch", [&] { b2.n++; kp.kernelParams = args; cudaGraphExecKernelNodeSetParams(ge, node, &kp); cudaGraphLaunch(ge, st); });
}
