// mma.sync m16n8k32 u8 x s8 -> s32 issue rate (per SMSP), 8 warps/SM, INDEP chains per warp.
#include <cstdio>
#include <cstdint>
template <int INDEP>
__global__ void k(int* out, int iters, long long* cyc) {
  int c[INDEP][4];
  for (int i = 0; i < INDEP; ++i) for (int e = 0; e < 4; ++e) c[i][e] = 0;
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 0x3c00, b1 = a0 ^ 0x3800;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < INDEP; ++i)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[i][0]), "+r"(c[i][1]), "+r"(c[i][2]), "+r"(c[i][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  long long t1 = clock64();
  int s = 0;
  for (int i = 0; i < INDEP; ++i) for (int e = 0; e < 4; ++e) s += c[i][e];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int INDEP>
void run(int warps) {
  int* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8);
  const int iters = 4096;
  k<INDEP><<<148, warps * 32>>>(out, iters, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per_warp = double(h) / (iters * INDEP);
  printf("IMMA k32 warps/SM %2d chains %d: %s %.2f cycles per IMMA per warp -> %.2f per SMSP\n", warps, INDEP, cudaGetErrorString(e),
         per_warp, per_warp / (warps / 4.0));
}
int main() {
  for (int w : {4, 8}) { run<1>(w); run<2>(w); run<4>(w); }
  return 0;
}
