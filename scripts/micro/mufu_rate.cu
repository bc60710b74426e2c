// Throughput of the FMHA softmax's inner loop on one SM: W warps, each
// running N iterations of 128 x (FFMA, ex2.approx, FADD) + 64 F2FP.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 mufu_rate.cu -o mufu_rate
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

template <int MODE>
__global__ void k(float* out, unsigned long long* cyc, int iters, float m) {
  float v[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) v[i] = (threadIdx.x + i) * 1e-3f;
  float s0 = 0, s1 = 0, s2 = 0, s3 = 0;
  unsigned acc = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 128; i += 2) {
      float a = fmaf(v[i], 1.4426950f, -m), b = fmaf(v[i + 1], 1.4426950f, -m);
      float pa, pb;
      if (MODE == 6) {            // f16x2 ex2, sums by mixed-precision adds, P already packed
        unsigned hx, hp;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hx) : "f"(b), "f"(a));
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(hp) : "r"(hx));
        acc ^= hp;
        float& sa = (i & 2) ? s2 : s0;
        float& sb = (i & 2) ? s3 : s1;
        asm volatile("{.reg .f16 lo, hi; mov.b32 {lo, hi}, %2; add.rn.f32.f16 %0, lo, %0; add.rn.f32.f16 %1, hi, %1;}"
                     : "+f"(sa), "+f"(sb) : "r"(hp));
        continue;
      }
      if (MODE == 5) {            // f16x2: pack x, one ex2 for two, unpack for the sums
        unsigned hx, hp;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hx) : "f"(b), "f"(a));
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(hp) : "r"(hx));
        acc ^= hp;
        asm volatile("{.reg .f16 lo, hi; mov.b32 {lo, hi}, %2; cvt.f32.f16 %0, lo; cvt.f32.f16 %1, hi;}"
                     : "=f"(pa), "=f"(pb) : "r"(hp));
      } else if (MODE == 4 && (i & 6) == 6) {   // 25 % on the FMA pipe (degree-3 polynomial)
        auto poly = [](float x) {
          x = fmaxf(x, -127.f);
          const float t = x + 12582912.f;
          const float f = x - (t - 12582912.f);
          float p = fmaf(f, 0.0551716685f, 0.242611155f);
          p = fmaf(p, f, 0.693260968f);
          p = fmaf(p, f, 0.999928057f);
          return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
        };
        pa = poly(a); pb = poly(b);
      } else if (MODE == 2) { pa = a; pb = b; }
      else {
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(pa) : "f"(a));
        asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(pb) : "f"(b));
      }
      if (i & 2) { s2 += pa; s3 += pb; } else { s0 += pa; s1 += pb; }
      if (MODE == 0 || MODE == 2 || MODE == 4) {
        unsigned r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(pb), "f"(pa));
        acc ^= r;
      } else if (MODE == 3) {     // round-half-up on the integer pipe: 2 IADD + PRMT
        unsigned r, ua = __float_as_uint(pa) + 0x8000u, ub = __float_as_uint(pb) + 0x8000u;
        asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r) : "r"(ua), "r"(ub));
        acc ^= r;
      }
    }
    m += 1e-7f;
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x % 32 == 0) cyc[blockIdx.x * 32 + threadIdx.x / 32] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2 + s3 + acc;
}

int main() {
  float* out; unsigned long long* cyc;
  cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 1 << 16);
  const int iters = 200;
  const char* names[] = {"ffma+ex2+fadd+f2fp", "ffma+ex2+fadd (no cvt)", "ffma+fadd+f2fp (no ex2)",
                         "ffma+ex2+fadd+int pack", "25% poly + f2fp", "f16x2 ex2 (no bf16 pack)",
                         "f16x2 ex2 + mixed adds"};
  for (int mode = 0; mode < 7; ++mode)
    for (int warps : {1, 2, 4, 8, 16}) {
      void (*f)(float*, unsigned long long*, int, float) =
          mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : mode == 3 ? k<3> : mode == 4 ? k<4> : mode == 5 ? k<5> : k<6>;
      f<<<1, warps * 32>>>(out, cyc, iters, 0.5f);
      f<<<1, warps * 32>>>(out, cyc, iters, 0.5f);
      cudaDeviceSynchronize();
      unsigned long long c[32];
      cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int w = 0; w < warps; ++w) mx = c[w] > mx ? c[w] : mx;
      double per_block = double(mx) / iters;   // cycles per 128-element block per warp
      double ex_per_clk_sm = 128.0 * 32 * warps * iters / mx;
      printf("%-26s warps %2d: %7.1f cycles per warp-block, %5.1f elements/clk/SM\n", names[mode], warps,
             per_block, ex_per_clk_sm);
    }
  return 0;
}
