// Microbenchmark of the decode GEMV inner loop (program.cu gemv_blocks) on shared-memory-resident
// synthetic tiles: cycles per 16x128 block per SM for W8 / W4 and variants, 8 consumer warps.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r; asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel)); return r;
}
template <bool VOL>
__device__ __forceinline__ void mma(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  if (VOL)
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  else
    asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// V: 0 = as program.cu, 1 = W4 with the OR constant in a register, 2 = no fold
template <int W, int NBLK, int V, bool VOL>
__device__ __forceinline__ void blocks(const uint8_t* blk, int bstride, const uint4* xl, int xstep, int kbstep,
                                       const float4* dxa, int dxstep, int lane, uint32_t c54, float (&y)[4]) {
  const int g = lane >> 2;
  const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
  float c[NBLK][4];
  for (int n = 0; n < NBLK; ++n) for (int e = 0; e < 4; ++e) c[n][e] = 0.f;
  if constexpr (W == 0) {
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int n = 0; n < NBLK; ++n) {
        const uint4 wv = reinterpret_cast<const uint4*>(blk + n * bstride)[p * 32 + lane];
        const uint4 xv = xl ? xl[n * kbstep + p * xstep] : z4;
        mma<VOL>(c[n], prmt(wv.x, 0x64646464u, 0x4140u), prmt(wv.x, 0x64646464u, 0x4342u), prmt(wv.y, 0x64646464u, 0x4140u),
                 prmt(wv.y, 0x64646464u, 0x4342u), xv.x, xv.y);
        mma<VOL>(c[n], prmt(wv.z, 0x64646464u, 0x4140u), prmt(wv.z, 0x64646464u, 0x4342u), prmt(wv.w, 0x64646464u, 0x4140u),
                 prmt(wv.w, 0x64646464u, 0x4342u), xv.z, xv.w);
      }
  } else {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int n = 0; n < NBLK; ++n) {
        const uint4 wv = reinterpret_cast<const uint4*>(blk + n * bstride)[i * 32 + lane];
        const uint4 x0 = xl ? xl[n * kbstep + (2 * i) * xstep] : z4;
        const uint4 x1 = xl ? xl[n * kbstep + (2 * i + 1) * xstep] : z4;
        const uint32_t qs[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t q = qs[u];
          const uint4 xv = u < 2 ? x0 : x1;
          if (V == 3) {
            // explicit lop3 (a & b) | c with both constants as immediates
            uint32_t r0, r1, r2, r3;
            asm("lop3.b32 %0, %1, 0x00F000F0, 0x54005400, 0xEA;" : "=r"(r0) : "r"(q << 4));
            asm("lop3.b32 %0, %1, 0x00F000F0, 0x54005400, 0xEA;" : "=r"(r1) : "r"(q >> 4));
            asm("lop3.b32 %0, %1, 0x00F000F0, 0x54005400, 0xEA;" : "=r"(r2) : "r"(q));
            asm("lop3.b32 %0, %1, 0x00F000F0, 0x54005400, 0xEA;" : "=r"(r3) : "r"(q >> 8));
            mma<VOL>(c[n], r0, r1, r2, r3, (u & 1) ? xv.z : xv.x, (u & 1) ? xv.w : xv.y);
          } else {
          const uint32_t C = V == 1 ? c54 : 0x54005400u;
          mma<VOL>(c[n], ((q << 4) & 0x00F000F0u) | C, ((q >> 4) & 0x00F000F0u) | C, (q & 0x00F000F0u) | C,
                   ((q >> 8) & 0x00F000F0u) | C, (u & 1) ? xv.z : xv.x, (u & 1) ? xv.w : xv.y);
          }
        }
      }
  }
  if (V == 2) {
    for (int n = 0; n < NBLK; ++n) for (int e = 0; e < 4; ++e) y[e] += c[n][e];
    return;
  }
  constexpr int cbytes = W == 0 ? 2048 : 1024;
#pragma unroll
  for (int n = 0; n < NBLK; ++n) {
    const uint8_t* bk = blk + n * bstride;
    const float s0 = *reinterpret_cast<const float*>(bk + cbytes + 4 * g);
    const float s1 = *reinterpret_cast<const float*>(bk + cbytes + 4 * (g + 8));
    const float z0 = __uint_as_float(0x4B000000u | bk[cbytes + 64 + g]) - 8388608.f;
    const float z1 = __uint_as_float(0x4B000000u | bk[cbytes + 64 + g + 8]) - 8388608.f;
    const float4 d = dxa[n * dxstep];
    const float D = W == 0 ? d.x : d.y;
    y[0] = fmaf(s0, c[n][0] - fmaf(z0, d.z, D), y[0]);
    y[2] = fmaf(s1, c[n][2] - fmaf(z1, d.z, D), y[2]);
  }
}
__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mb_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(su32(bar)), "r"(parity) : "memory");
  } while (!ok);
}
__device__ __forceinline__ void mb_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(bar)) : "memory");
}
template <int W, int V, bool VOL, int RING, int NB = 2>
__global__ void __launch_bounds__(288, 1) k(float* out, int reps, long long* cyc) {
  extern __shared__ __align__(16) uint8_t sm[];
  constexpr int bsz = W == 0 ? 2128 : 1104, nb = W == 0 ? 16 : 32;
  uint4* xs = reinterpret_cast<uint4*>(sm + 40000);
  float4* dx = reinterpret_cast<float4*>(sm + 40000 + 32 * 4 * 4 * 16);
  for (int i = threadIdx.x; i < 40000 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  for (int i = threadIdx.x; i < 32 * 16; i += blockDim.x) xs[i] = make_uint4(0x3c003c00u, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u);
  for (int i = threadIdx.x; i < 64; i += blockDim.x) dx[i] = make_float4(1.f, 1.f, 1.f, 0.f);
  __shared__ uint64_t full[5], empty[5];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 5; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[i])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[i])), "r"(8));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (RING && warp == 8) {
    if (lane == 0) {
      int si = 0; uint32_t ph = 0;
      for (int r = 0; r < reps; ++r) {
        mb_wait(&empty[si], ph ^ 1u);
        mb_arrive(&full[si]);
        if (++si == 5) { si = 0; ph ^= 1u; }
      }
    }
  }
  uint32_t c54 = static_cast<uint32_t>(reps) * 0u + 0x54005400u;
  asm volatile("" : "+r"(c54));  // opaque to ptxas? (reps is a runtime value)
  c54 = reps > 0 ? c54 ^ static_cast<uint32_t>(reps >> 30) : c54;
  float y[4] = {0.f, 0.f, 0.f, 0.f};
  long long t0 = clock64();
  if (warp < 8) {
    const int g = lane >> 2, tig = lane & 3;
    const uint4* xl = g < 1 ? xs + tig : nullptr;
    int si = 0; uint32_t ph = 0;
    for (int r = 0; r < reps; ++r) {
      if (RING) mb_wait(&full[si], ph);
      for (int j = warp; j < nb; j += 8 * NB) {
        const uint8_t* bk = sm + j * bsz;
        blocks<W, NB, V, VOL>(bk, 8 * bsz, xl ? xl + j * 16 : nullptr, 4, 8 * 16, dx + j, 8, lane, c54, y);
      }
      __syncwarp();
      if (RING) {
        if (lane == 0) mb_arrive(&empty[si]);
        if (++si == 5) { si = 0; ph ^= 1u; }
      }
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = y[0] + y[1] + y[2] + y[3];
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int W, int V, bool VOL, int RING = 0, int NB = 2>
void run(const char* name) {
  float* out; long long* cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 8);
  const int reps = 2000, smem = 60000;
  cudaFuncSetAttribute(k<W, V, VOL, RING, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<W, V, VOL, RING, NB><<<148, 288, smem>>>(out, reps, cyc);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<W, V, VOL, RING, NB><<<148, 288, smem>>>(out, reps, cyc);
  cudaEventRecord(e1);
  cudaError_t e = cudaDeviceSynchronize();
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("  [%s] %.2f ns per block per SM (wall), ", name, ms * 1e6 / (reps * (W == 0 ? 16 : 32)));
  long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const int nb = W == 0 ? 16 : 32;
  printf("%-28s %s: %.1f cycles per block per SM (%.1f codes/cycle/SM)\n", name, cudaGetErrorString(e), double(h) / (reps * nb),
         2048.0 * reps * nb / double(h));
}
int main() {
  run<0, 0, true>("W8 base");
  run<0, 2, true>("W8 no fold");
  run<0, 0, false>("W8 nonvolatile mma");
  run<1, 0, true>("W4 base");
  run<1, 1, true>("W4 reg const");
  run<1, 2, true>("W4 no fold");
  run<1, 1, false>("W4 reg const nonvolatile");
  run<0, 0, true, 1>("W8 base + ring protocol");
  run<0, 0, true, 0, 1>("W8 NBLK=1");
  run<1, 0, true, 0, 4>("W4 NBLK=4");
  run<1, 1, true, 0, 4>("W4 NBLK=4 reg const");
  run<1, 3, true>("W4 lop3 asm");
  run<1, 0, true, 1>("W4 base + ring protocol");
  return 0;
}
