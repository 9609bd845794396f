// peaks.cu -- INT32 issue-rate microbenchmarks: the roofline denominator for this path.
// MEASURED_PEAKS.json only carries HBM and bf16 numbers; Dilithium's hot loops are
// LOP3/SHF (Keccak, alu pipe) and IMAD (Montgomery NTT, fma pipe), so the engine measures
// those rates itself, live, on the device it runs on.
#include "engine.cuh"

namespace dlb {

template <int MODE>
__global__ void __launch_bounds__(256) k_peak_int32(uint32_t* out, int iters, uint32_t seed) {
  uint32_t x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = seed + threadIdx.x * 8 + i;
  const uint32_t a = seed | 1u, b = seed ^ 0x9e3779b9u;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int rep = 0; rep < 8; ++rep) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (MODE == 0) {
          asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(a), "r"(b));
        } else if (MODE == 1) {
          asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
        } else if (MODE == 2) {
          asm volatile("shf.l.wrap.b32 %0, %0, %1, 7;" : "+r"(x[i]) : "r"(x[(i + 1) & 7]));
        } else if (MODE == 3) {
          if (i & 1) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[i]) : "r"(a), "r"(b));
          else asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
        } else if (MODE == 4) {
          asm volatile("mul.hi.s32 %0, %0, %1;" : "+r"(x[i]) : "r"(a));
        } else {
          asm volatile("{ .reg .b64 t; mul.wide.s32 t, %0, %1; mov.b64 {%0, _}, t; }" : "+r"(x[i]) : "r"(a));
        }
      }
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc ^= x[i];
  if (acc == 0x12345678u) out[0] = acc;  // keeps the chain live without a store per thread
}

template <int MODE>
static int run_peak(dlb_ctx* c, uint32_t* scratch, double* tops) {
  const int iters = 2048;
  const int grid = c->sm_count * 8;
  cudaStream_t st = c->s();
  k_peak_int32<MODE><<<grid, 256, 0, st>>>(scratch, 64, 1u);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(c->ev0, st);
    k_peak_int32<MODE><<<grid, 256, 0, st>>>(scratch, iters, 3u + rep);
    cudaEventRecord(c->ev1, st);
    DLB_CUDA_CHECK(cudaStreamSynchronize(st));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev0, c->ev1);
    if (ms < best) best = ms;
  }
  const double ops = (double)grid * 256.0 * iters * 64.0;
  *tops = ops / (best * 1e-3) / 1e12;
  return 0;
}

}  // namespace dlb

// out[0] LOP3, out[1] IMAD, out[2] SHF, out[3] LOP3+IMAD interleaved; in 10^12 lane-ops/s
extern "C" int dlb_measure_int32_peak(dlb_ctx* c, double* out) {
  if (!c || !out) return DLB_E_ARG;
  cudaSetDevice(c->device);
  uint32_t* scratch;
  DLB_TRY(dlb::dalloc(c, "peak", 64, &scratch));
  DLB_TRY(dlb::run_peak<0>(c, scratch, &out[0]));
  DLB_TRY(dlb::run_peak<1>(c, scratch, &out[1]));
  DLB_TRY(dlb::run_peak<2>(c, scratch, &out[2]));
  DLB_TRY(dlb::run_peak<3>(c, scratch, &out[3]));
  return 0;
}

// out[0] mul.hi.s32 (IMAD.HI), out[1] mul.wide.s32 (IMAD.WIDE): the Montgomery-product
// building blocks, same unit as above
extern "C" int dlb_measure_imad_hi_peak(dlb_ctx* c, double* out) {
  if (!c || !out) return DLB_E_ARG;
  cudaSetDevice(c->device);
  uint32_t* scratch;
  DLB_TRY(dlb::dalloc(c, "peak", 64, &scratch));
  DLB_TRY(dlb::run_peak<4>(c, scratch, &out[0]));
  DLB_TRY(dlb::run_peak<5>(c, scratch, &out[1]));
  return 0;
}
