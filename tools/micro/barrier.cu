// Grid-barrier latency on B200 (148 CTAs x 384 threads, one per SM): microseconds per barrier for
// (0) fence + atomicAdd + acquire poll, (1) release reduction + relaxed poll + acquire fence,
// (2) two-level: 8-CTA group counters, the group's last arriver bumps the global counter.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) { unsigned v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) { unsigned v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v; }
template <int V>
__global__ void __launch_bounds__(384, 1) k(unsigned* ctr, int reps, unsigned long long* out) {
  unsigned epoch = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    __syncthreads();
    if (threadIdx.x == 0) {
      ++epoch;
      if (V == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        while (ld_acq(ctr) < epoch * gridDim.x) {}
        __threadfence();
      } else if (V == 1) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        while (ld_rlx(ctr) < epoch * gridDim.x) {}
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      } else {
        const unsigned ng = (gridDim.x + 7) / 8, g = blockIdx.x / 8;
        const unsigned gsz = min(8u, gridDim.x - g * 8);
        unsigned old;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(ctr + 32 * (1 + g)), "r"(1) : "memory");
        if (old + 1 == epoch * gsz) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        while (ld_rlx(ctr) < epoch * ng) {}
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
    }
    __syncthreads();
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = t1 - t0;
}
template <int V>
void run(const char* name) {
  unsigned* ctr; unsigned long long* out;
  cudaMalloc(&ctr, 64 * 1024); cudaMalloc(&out, 8);
  const int reps = 2000;
  for (int it = 0; it < 2; ++it) {
    cudaMemset(ctr, 0, 64 * 1024);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k<V><<<148, 384>>>(ctr, reps, out);
    cudaEventRecord(b);
    cudaError_t e = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (it == 1) printf("%-34s %s: %.3f us per barrier\n", name, cudaGetErrorString(e), ms * 1e3 / reps);
  }
}
int main() {
  run<0>("fence + atomicAdd + acquire poll");
  run<1>("release red + relaxed poll + fence");
  run<2>("two-level (8-CTA groups)");
  return 0;
}
