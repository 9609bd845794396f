// Do the two instruction families of the signing path overlap when they run in DIFFERENT warps of
// one SM sub-partition?  Role K = the kernel's Keccak-f[1600] (LOP3 / SHF, alu pipe); role B =
// the kernel's forward + inverse NTT (IMAD.HI + 2 IMAD + add / sub, shared-memory transposes).
// Every block (4 warps = one warp per sub-partition) loops its role for a fixed time window and
// counts iterations, so all resident warps are active for the whole measurement.  Compared:
// W warps per sub-partition all K, all B, and half / half.  If the mixed run keeps each role near
// its solo per-warp rate, the stages of the scheduler kernel can overlap; if each role drops to
// half, the sub-partition is issue-bound and stage overlap buys nothing.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/coissue scripts/ubench/coissue.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../paper_2211_12265_b200/csrc/keccak.cuh"
#include "../../paper_2211_12265_b200/csrc/ntt.cuh"

using namespace dlb;

__global__ void __launch_bounds__(128) k_roles(int mix, int sms, unsigned long long window_ns,
                                               unsigned long long* counts, uint32_t* sink) {
  __shared__ __align__(16) int2 zs[256], nzs[256];
  __shared__ __align__(16) int32_t tiles[4][kTileWords];
  load_twiddles(zs, nzs);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // mix: 0 all K, 1 all B, 2 alternate by resident wave so every SM holds both roles
  const int role = mix == 2 ? (int)((blockIdx.x / sms) & 1) : mix;
  unsigned long long t0, now;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  unsigned long long iters = 0;
  uint32_t acc = 0;
  if (role == 0) {
    uint64_t s[25];
#pragma unroll
    for (int i = 0; i < 25; ++i) s[i] = (uint64_t)(threadIdx.x + 1) * 0x9E3779B97F4A7C15ull + i;
    do {
#pragma unroll 1
      for (int r = 0; r < 4; ++r) keccak_f1600(s);
      iters += 4;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    } while (now - t0 < window_ns);
    acc = (uint32_t)s[0] ^ (uint32_t)s[7];
  } else {
    int32_t r8[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) r8[i] = (int32_t)(threadIdx.x * 8 + i) % kQ;
    do {
#pragma unroll 1
      for (int r = 0; r < 4; ++r) {
        ntt_fwd(r8, tiles[warp], zs, lane);
#pragma unroll
        for (int i = 0; i < 8; ++i) r8[i] = reduce32(r8[i]);
        ntt_inv(r8, tiles[warp], nzs, lane);
      }
      iters += 4;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    } while (now - t0 < window_ns);
    acc = (uint32_t)r8[0] ^ (uint32_t)r8[5];
  }
  if (lane == 0) atomicAdd(&counts[role], iters);
  if (acc == 0x12345678u) sink[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* counts;
  uint32_t* sink;
  cudaMalloc(&counts, 16);
  cudaMalloc(&sink, 64);
  const unsigned long long window = 3000000ull;  // 3 ms
  printf("role K = keccak_f1600 (one sponge per thread), role B = ntt_fwd + ntt_inv (one warp per polynomial)\n");
  printf("rates per WARP in kilo-iterations/s (K: permutation calls, B: forward+inverse pairs)\n");
  for (int wps : {2, 4, 8}) {
    double solo[2] = {0, 0};
    for (int mix = 0; mix < 3; ++mix) {
      cudaMemset(counts, 0, 16);
      k_roles<<<sms * wps, 128>>>(mix, sms, window, counts, sink);
      cudaDeviceSynchronize();
      unsigned long long h[2];
      cudaMemcpy(h, counts, 16, cudaMemcpyDeviceToHost);
      const double warpsK = mix == 0 ? sms * wps * 4.0 : (mix == 2 ? sms * wps * 2.0 : 0);
      const double warpsB = mix == 1 ? sms * wps * 4.0 : (mix == 2 ? sms * wps * 2.0 : 0);
      const double rk = warpsK ? h[0] / warpsK / (window * 1e-9) / 1e3 : 0;
      const double rb = warpsB ? h[1] / warpsB / (window * 1e-9) / 1e3 : 0;
      if (mix == 0) solo[0] = rk;
      if (mix == 1) solo[1] = rb;
      if (mix < 2)
        printf("warps/SMSP %d  all %s: %.1f per warp  (SM total %.0f)\n", wps, mix == 0 ? "K" : "B", mix == 0 ? rk : rb,
               (mix == 0 ? rk : rb) * wps * 4);
      else
        // a time-sliced SM (half the time all K, half all B) gives each role 0.5 x W x solo; the
        // mixed run gives (W/2) x rate: the ratio rate / solo is the gain over time slicing, 1 .. 2
        printf("warps/SMSP %d  half K + half B: K %.1f per warp = x%.2f, B %.1f per warp = x%.2f of the solo "
               "per-warp rate (1.0 = no better than running the stages one after the other, 2.0 = full overlap)\n",
               wps, rk, rk / solo[0], rb, rb / solo[1]);
    }
  }
  return 0;
}
