// Microbenchmark: issue rate of mma.sync.m16n8k16 f16->f32 on one SM (8 warps), with INDEP
// independent accumulator chains per warp.  Prints cycles per HMMA per SM sub-partition.
#include <cstdio>
#include <cstdint>
template <int INDEP>
__global__ void k(float* out, int iters, long long* cyc) {
  float c[INDEP][4];
  for (int i = 0; i < INDEP; ++i) for (int e = 0; e < 4; ++e) c[i][e] = 0.f;
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x3c00, b1 = a0 ^ 0x3800;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < INDEP; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int i = 0; i < INDEP; ++i) for (int e = 0; e < 4; ++e) s += c[i][e];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int INDEP>
void run(int warps) {
  float* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8);
  const int iters = 4096;
  k<INDEP><<<148, warps * 32>>>(out, iters, cyc);
  cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_warp = double(h) / (iters * INDEP);  // cycles per HMMA per warp
  printf("warps/SM %2d chains %d: %.2f cycles per HMMA per warp -> %.2f cycles per HMMA per SMSP\n", warps, INDEP,
         per_warp, per_warp / (warps / 4.0));
  cudaFree(out); cudaFree(cyc);
}
int main() {
  for (int w : {4, 8, 16}) { run<1>(w); run<2>(w); run<4>(w); run<8>(w); }
  return 0;
}
