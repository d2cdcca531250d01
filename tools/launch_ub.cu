#include <cstdio>
#include <chrono>
#include <cuda_runtime.h>
struct Big { const double* a; const unsigned long long* b; size_t n, ld; unsigned long long s; double dt; void* o; void* f; unsigned* c; double* fs; volatile unsigned* ff; };
__global__ void k_small(int x) { if (x == 12345) printf("x"); }
__global__ void k_big(Big b) { if (b.n == 12345) printf("x"); }
int main() {
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  Big b{}; 
  for (int rep = 0; rep < 2; ++rep) {
    for (int which = 0; which < 2; ++which) {
      cudaStreamSynchronize(st);
      auto t0 = std::chrono::steady_clock::now();
      for (int i = 0; i < 1000; ++i) { if (which) k_big<<<512, 32, 0, st>>>(b); else k_small<<<512, 32, 0, st>>>(i); }
      auto t1 = std::chrono::steady_clock::now();
      cudaStreamSynchronize(st);
      auto t2 = std::chrono::steady_clock::now();
      double l = std::chrono::duration<double, std::micro>(t1 - t0).count() / 1000;
      // launch + sync round trip
      double rt = 0;
      for (int i = 0; i < 200; ++i) {
        auto a = std::chrono::steady_clock::now();
        if (which) k_big<<<512, 32, 0, st>>>(b); else k_small<<<512, 32, 0, st>>>(i);
        cudaStreamSynchronize(st);
        rt += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - a).count();
      }
      printf("%s: launch %.2f us/launch (queued), launch+sync round trip %.2f us\n", which ? "big args" : "small args", l, rt / 200);
    }
  }
}
