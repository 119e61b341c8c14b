// Per-SM throughput of the instructions in the softmax inner loop (one CTA/SM, 4..16 warps).
#include <cstdio>
#include <cuda_bf16.h>
#define N_ITER 4096
template <int OP>
__global__ void k(float* out, float a, float b, long long* cyc) {
  float x0 = a + threadIdx.x, x1 = b - threadIdx.x, x2 = a * 0.5f, x3 = b * 0.25f;
  float y0 = 0, y1 = 0, y2 = 0, y3 = 0;
  unsigned u0 = 0x3c003c00u ^ threadIdx.x, u1 = 0xbc00bc00u, v0 = 0x3f803f80u, v1 = 0xbf00bf00u;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < N_ITER; ++i) {
    if (OP == 0) {  // MUFU.EX2 x4 independent
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x1));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x2)); asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x3));
    } else if (OP == 1) {  // FFMA2 x2 (4 fmas)
      asm volatile("{.reg .b64 a,b; mov.b64 a,{%0,%1}; mov.b64 b,{%2,%3}; fma.rn.f32x2 a,a,b,b; mov.b64 {%0,%1},a;}" : "+f"(x0), "+f"(x1) : "f"(x2), "f"(x3));
      asm volatile("{.reg .b64 a,b; mov.b64 a,{%0,%1}; mov.b64 b,{%2,%3}; fma.rn.f32x2 a,a,b,b; mov.b64 {%0,%1},a;}" : "+f"(y0), "+f"(y1) : "f"(x2), "f"(x3));
    } else if (OP == 2) {  // FFMA x4
      asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(x0) : "f"(x2)); asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(x1) : "f"(x3));
      asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(y0) : "f"(x2)); asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(y1) : "f"(x3));
    } else if (OP == 3) {  // FADD2 x2
      asm volatile("{.reg .b64 a,b; mov.b64 a,{%0,%1}; mov.b64 b,{%2,%3}; add.rn.f32x2 a,a,b; mov.b64 {%0,%1},a;}" : "+f"(x0), "+f"(x1) : "f"(x2), "f"(x3));
      asm volatile("{.reg .b64 a,b; mov.b64 a,{%0,%1}; mov.b64 b,{%2,%3}; add.rn.f32x2 a,a,b; mov.b64 {%0,%1},a;}" : "+f"(y0), "+f"(y1) : "f"(x2), "f"(x3));
    } else if (OP == 4) {  // FMNMX3 x4
      asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(x0) : "f"(x2), "f"(x3)); asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(x1) : "f"(x2), "f"(x3));
      asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(y0) : "f"(x2), "f"(x3)); asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(y1) : "f"(x2), "f"(x3));
    } else if (OP == 5) {  // F2FP bf16x2 pack x4
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u0) : "f"(x0), "f"(x1)); asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u1) : "f"(x2), "f"(x3));
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u0) : "f"(x1), "f"(x0)); asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u1) : "f"(x3), "f"(x2));
      x0 += 1.0f;
    } else if (OP == 6) {  // mix: 1 MUFU + 1 FFMA2 + 1 FADD2 + 1 F2FP  (softmax pair body / 2)
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x0));
      asm volatile("{.reg .b64 a,b; mov.b64 a,{%0,%1}; mov.b64 b,{%2,%3}; fma.rn.f32x2 a,a,b,b; mov.b64 {%0,%1},a;}" : "+f"(y0), "+f"(y1) : "f"(x2), "f"(x3));
      asm volatile("{.reg .b64 a,b; mov.b64 a,{%0,%1}; mov.b64 b,{%2,%3}; add.rn.f32x2 a,a,b; mov.b64 {%0,%1},a;}" : "+f"(y2), "+f"(y3) : "f"(x2), "f"(x3));
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u0) : "f"(x1), "f"(x2));
      x1 += 0.5f;
    } else if (OP == 7) {  // ex2.approx.f16x2 x4 (2 results each)
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u0)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u1));
      asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v0)); asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v1));
    } else if (OP == 8) {  // ex2.approx.ftz.bf16x2 x4 (2 results each)
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u0)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u1));
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v0)); asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v1));
    } else if (OP == 9) {  // bf16x2 softmax pair body: FFMA2, F2FP pack, EX2.bf16x2, 2x unpack, FADD2
      asm volatile("{.reg .b64 a,b; mov.b64 a,{%0,%1}; mov.b64 b,{%2,%3}; fma.rn.f32x2 a,a,b,b; mov.b64 {%0,%1},a;}" : "+f"(x0), "+f"(x1) : "f"(x2), "f"(x3));
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u0) : "f"(x1), "f"(x0));
      asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u0));
      float lo = __uint_as_float(u0 << 16), hi = __uint_as_float(u0 & 0xffff0000u);
      asm volatile("{.reg .b64 a,b; mov.b64 a,{%0,%1}; mov.b64 b,{%2,%3}; add.rn.f32x2 a,a,b; mov.b64 {%0,%1},a;}" : "+f"(y0), "+f"(y1) : "f"(lo), "f"(hi));
      v0 ^= u0;
      x0 += 0.5f;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + y0 + y1 + y2 + y3 + u0 + u1 + v0 + v1;
}
int main() {
  float* out; long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const char* names[] = {"MUFU.EX2", "FFMA2 (2 fma each)", "FFMA", "FADD2 (2 add each)", "FMNMX3", "F2FP.BF16 pack", "mix (EX2+FFMA2+FADD2+F2FP)",
                         "EX2.f16x2 (2 exp each)", "EX2.bf16x2 (2 exp each)", "bf16x2 pair body (6 instr)"};
  const int per_iter[] = {4, 2, 4, 2, 4, 4, 4, 4, 4, 1};
  for (int warps : {4, 8, 12, 16}) {
    for (int op = 0; op < 10; ++op) {
      auto run = [&](auto kern) { kern<<<148, warps * 32>>>(out, 0.1f, 0.2f, cyc); };
      switch (op) { case 0: run(k<0>); break; case 1: run(k<1>); break; case 2: run(k<2>); break;
                    case 3: run(k<3>); break; case 4: run(k<4>); break; case 5: run(k<5>); break; case 6: run(k<6>); break;
                    case 7: run(k<7>); break; case 8: run(k<8>); break; case 9: run(k<9>); break; }
      cudaDeviceSynchronize();
      long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
      double instr_per_smsp = (double)N_ITER * per_iter[op] * warps / 4.0;
      printf("warps=%2d %-28s %6.2f cycles per warp-instruction per SMSP\n", warps, names[op], c / instr_per_smsp);
    }
  }
  return 0;
}
