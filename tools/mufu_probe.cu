// Throughput of ex2.approx (MUFU) vs FFMA vs the poly_exp2 emulation per SM (timing only).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float poly(float x) {
  x = fmaxf(x, -127.0f);
  const float t = x + 12582912.0f;
  const float f = x - (t - 12582912.0f);
  const float p = fmaf(fmaf(fmaf(0.05500893f, f, 0.24221101f), f, 0.69328293f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
template <int MODE>
__global__ void k(float* out, int iters, long long* cyc) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) a[i] = ex2(a[i]) - 1.5f;
      else if (MODE == 1) a[i] = fmaf(a[i], 0.999f, -0.001f);
      else a[i] = poly(a[i]) - 1.5f;
    }
  }
  long long t1 = clock64();
  float s = 0; for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const char* names[3] = {"ex2 (+FADD)", "FFMA", "poly_exp2 (+FADD)"};
  for (int warps = 4; warps <= 32; warps *= 2) {
    for (int mode = 0; mode < 3; ++mode) {
      const int iters = 256;
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) k<0><<<148, warps * 32>>>(out, iters, cyc);
        if (mode == 1) k<1><<<148, warps * 32>>>(out, iters, cyc);
        if (mode == 2) k<2><<<148, warps * 32>>>(out, iters, cyc);
      }
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      const double per_sm = (double)warps * 32 * iters * 16 / c;
      printf("warps/SM %2d %-18s: %.1f results/clk/SM (%.2f cyc per warp-op per SMSP)\n", warps, names[mode], per_sm,
             32.0 * 4 / per_sm);
    }
  }
  return 0;
}
