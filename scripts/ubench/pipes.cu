// Pipe co-issue microbenchmarks for the Montgomery butterfly / Keccak instruction mix.
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pipes scripts/ubench/pipes.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kQ = 8380417;

template <int MODE>
__global__ void __launch_bounds__(128) k(uint32_t* out, int iters, uint32_t seed) {
  int32_t x[8];
  uint32_t y[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { x[i] = seed + threadIdx.x * 8 + i; y[i] = seed * 3 + i; }
  const int32_t a = seed | 1u, b = seed ^ 0x9e3779b9u;
  const uint32_t ua = a, ub = b;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int rep = 0; rep < 4; ++rep) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (MODE == 0) {  // LOP3 only (2 per slot)
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[i]) : "r"(ua), "r"(ub));
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[i]) : "r"(ub), "r"(ua));
        } else if (MODE == 1) {  // IMAD lo + LOP3
          asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[i]) : "r"(ua), "r"(ub));
        } else if (MODE == 2) {  // IMAD.WIDE (both halves live) + LOP3
          asm volatile("{ .reg .b64 t; .reg .b32 lo, hi; mul.wide.s32 t, %0, %1; mov.b64 {lo, hi}, t; xor.b32 %0, lo, hi; }" : "+r"(x[i]) : "r"(a));
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[i]) : "r"(ua), "r"(ub));
        } else if (MODE == 3) {  // IMAD.HI + LOP3
          asm volatile("mul.hi.s32 %0, %0, %1;" : "+r"(x[i]) : "r"(a));
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[i]) : "r"(ua), "r"(ub));
        } else if (MODE == 4) {  // two IMAD.HI
          asm volatile("mul.hi.s32 %0, %0, %1;" : "+r"(x[i]) : "r"(a));
          asm volatile("mul.hi.s32 %0, %0, %1;" : "+r"(x[i]) : "r"(b));
        } else if (MODE == 5) {  // Montgomery butterfly as compiled today (5 instr) alone
          int32_t t;
          asm volatile("mul.lo.s32 %0, %1, %2;" : "=r"(t) : "r"(x[i]), "r"(b));
          int64_t w;
          asm volatile("mul.wide.s32 %0, %1, %2;" : "=l"(w) : "r"(t), "r"(-kQ));
          int32_t h;
          asm volatile("{ .reg .b64 p; mad.wide.s32 p, %1, %2, %3; mov.b64 {_, %0}, p; }" : "=r"(h) : "r"(x[i]), "r"(a), "l"(w));
          const int32_t u = x[(i + 4) & 7];
          x[i] = u + h;
          x[(i + 4) & 7] = u - h;
        } else if (MODE == 6) {  // same butterfly + 5 LOP3 (Keccak-like co-runner in the same warp)
          int32_t t;
          asm volatile("mul.lo.s32 %0, %1, %2;" : "=r"(t) : "r"(x[i]), "r"(b));
          int64_t w;
          asm volatile("mul.wide.s32 %0, %1, %2;" : "=l"(w) : "r"(t), "r"(-kQ));
          int32_t h;
          asm volatile("{ .reg .b64 p; mad.wide.s32 p, %1, %2, %3; mov.b64 {_, %0}, p; }" : "=r"(h) : "r"(x[i]), "r"(a), "l"(w));
          const int32_t u = x[(i + 4) & 7];
          x[i] = u + h;
          x[(i + 4) & 7] = u - h;
#pragma unroll
          for (int q = 0; q < 5; ++q)
            asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[i]) : "r"(ua), "r"(ub));
        } else if (MODE == 7) {  // 64-bit accumulate IMAD.WIDE alone
          int64_t acc = ((int64_t)x[i] << 32) | y[i];
          asm volatile("mad.wide.s32 %0, %1, %2, %0;" : "+l"(acc) : "r"(a), "r"(b));
          asm volatile("mad.wide.s32 %0, %1, %2, %0;" : "+l"(acc) : "r"(b), "r"(a));
          x[i] = (int32_t)(acc >> 32); y[i] = (uint32_t)acc;
        } else if (MODE == 8) {  // SHF + LOP3 (Keccak mix)
          asm volatile("shf.l.wrap.b32 %0, %0, %1, 7;" : "+r"(y[i]) : "r"(y[(i + 1) & 7]));
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[i]) : "r"(ua), "r"(ub));
        } else if (MODE == 10 || MODE == 11) {  // Shoup-style butterfly: HI(a,w'), lo(a*w), lo(h*-q + .), add, sub
          int32_t h, t;
          asm volatile("mul.hi.s32 %0, %1, %2;" : "=r"(h) : "r"(x[i]), "r"(b));
          asm volatile("mul.lo.s32 %0, %1, %2;" : "=r"(t) : "r"(x[i]), "r"(a));
          asm volatile("mad.lo.s32 %0, %1, %2, %0;" : "+r"(t) : "r"(h), "r"(-kQ));
          const int32_t u = x[(i + 4) & 7];
          x[i] = u + t;
          x[(i + 4) & 7] = u - t;
          if (MODE == 11) {
#pragma unroll
            for (int q = 0; q < 5; ++q)
              asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(y[i]) : "r"(ua), "r"(ub));
          }
        } else if (MODE == 12) {  // LOP3 with three distinct register operands (Keccak-like)
          asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(y[i]) : "r"(y[(i + 1) & 7]), "r"(y[(i + 3) & 7]), "r"(y[(i + 5) & 7]));
          asm volatile("lop3.b32 %0, %1, %2, %3, 0xd2;" : "=r"(y[(i + 2) & 7]) : "r"(y[(i + 4) & 7]), "r"(y[(i + 6) & 7]), "r"(y[(i + 7) & 7]));
        } else if (MODE == 9) {  // IADD3 + IMAD lo
          asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
          asm volatile("add.s32 %0, %0, %1;" : "+r"(y[i]) : "r"(ua));
        }
      }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc ^= (uint32_t)x[i] ^ y[i];
  if (acc == 0x12345678u) out[0] = acc;
}

template <int MODE>
void run(const char* name, double inst_per_slot, int wps) {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  uint32_t* out;
  cudaMalloc(&out, 64);
  const int iters = 4096;
  const int grid = sms * wps;  // wps blocks of 4 warps per SM -> wps warps per SMSP
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<grid, 128>>>(out, 64, 1u);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    k<MODE><<<grid, 128>>>(out, iters, 3u + r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double warp_inst = (double)grid * 4 * iters * 32.0 * inst_per_slot;
  const double ipc = warp_inst / (best * 1e-3) / (clk * 1e3) / (sms * 4.0);
  printf("%-34s warps/SMSP %2d  IPC/SMSP %.3f  (%.3f ms)\n", name, wps, ipc, best);
  cudaFree(out);
}

int main() {
  for (int wps : {1, 4}) {
    run<0>("LOP3 x2", 2, wps);
    run<1>("IMAD.lo + LOP3", 2, wps);
    run<2>("IMAD.WIDE(+xor) + LOP3", 3, wps);
    run<3>("IMAD.HI + LOP3", 2, wps);
    run<4>("IMAD.HI x2", 2, wps);
    run<5>("butterfly (IMAD,WIDE,HI,add,sub)", 5, wps);
    run<6>("butterfly + 5 LOP3", 10, wps);
    run<7>("IMAD.WIDE acc64 x2", 2, wps);
    run<8>("SHF + LOP3", 2, wps);
    run<9>("IMAD.lo + IADD", 2, wps);
    run<10>("shoup butterfly (HI,lo,lo,add,sub)", 5, wps);
    run<11>("shoup butterfly + 5 LOP3", 10, wps);
    run<12>("LOP3 x2 distinct regs", 2, wps);
  }
  return 0;
}
