// A/B evidence for two thread mappings this engine does NOT use:
//   (1) Keccak-f[1600] with ONE state spread over 25 lanes of a warp (the paper's mapping:
//       theta / chi neighbours by shuffles) against one state per thread (keccak.cuh);
//   (2) the forward NTT with its five short-distance levels done by warp shuffles against
//       the register passes + two shared-memory transposes of ntt.cuh.
// Both variants are checked bit for bit against the engine's routines before they are timed.
// build: nvcc -O3 -std=c++17 --expt-relaxed-constexpr -gencode arch=compute_100a,code=sm_100a -o /tmp/mapping_ab scripts/ubench/mapping_ab.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "../../paper_2211_12265_b200/csrc/keccak.cuh"
#include "../../paper_2211_12265_b200/csrc/ntt.cuh"

using namespace dlb;

// ---- (1) warp-cooperative Keccak: lane x + 5 y holds A[x][y]; lanes 25..31 idle ------------
__device__ __constant__ int kRho[25] = {0, 1, 62, 28, 27, 36, 44, 6, 55, 20, 3, 10, 43, 25, 39,
                                        41, 45, 15, 21, 8, 18, 2, 61, 56, 14};
__device__ __forceinline__ uint64_t shfl64(uint64_t v, int src) {
  const uint32_t lo = __shfl_sync(0xffffffffu, (uint32_t)v, src);
  const uint32_t hi = __shfl_sync(0xffffffffu, (uint32_t)(v >> 32), src);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t rotl64v(uint64_t x, int r) {
  return r ? (x << r) | (x >> (64 - r)) : x;
}
__device__ __forceinline__ uint64_t keccak_coop(uint64_t a, int lane) {
  const int l = lane < 25 ? lane : 0, x = l % 5, y = l / 5;
  // pi: B[y][2x+3y] = rot(A[x][y]); the lane that ends up holding B[X][Y] reads from x' with
  // X = y', Y = 2x'+3y'  ->  x' = (X + 3Y) % 5, y' = X
  const int src = ((x + 3 * y) % 5) + 5 * x;
  const int rho = kRho[src];
#pragma unroll 1
  for (int r = 0; r < 24; ++r) {
    // theta: column parity by four shuffles, then D from the two neighbour columns
    uint64_t c = a;
#pragma unroll
    for (int k = 1; k < 5; ++k) c ^= shfl64(a, x + 5 * ((y + k) % 5));
    const uint64_t d = shfl64(c, (x + 4) % 5) ^ rotl64v(shfl64(c, (x + 1) % 5), 1);
    a ^= d;
    // rho + pi
    const uint64_t b = rotl64v(shfl64(a, src), rho);
    // chi
    const uint64_t b1 = shfl64(b, (x + 1) % 5 + 5 * y), b2 = shfl64(b, (x + 2) % 5 + 5 * y);
    a = b ^ (~b1 & b2);
    if (lane == 0) a ^= kKeccakRC[r];
  }
  return a;
}

__global__ void k_keccak_thread(uint64_t* states, int perms) {
  uint64_t s[25];
  const size_t t = blockIdx.x * blockDim.x + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 25; ++i) s[i] = states[t * 25 + i];
#pragma unroll 1
  for (int p = 0; p < perms; ++p) keccak_f1600(s);
#pragma unroll
  for (int i = 0; i < 25; ++i) states[t * 25 + i] = s[i];
}
__global__ void k_keccak_coop(uint64_t* states, int perms) {  // one state per WARP
  const int lane = threadIdx.x & 31;
  const size_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint64_t a = lane < 25 ? states[w * 25 + lane] : 0;
#pragma unroll 1
  for (int p = 0; p < perms; ++p) a = keccak_coop(a, lane);
  if (lane < 25) states[w * 25 + lane] = a;
}

// ---- (2) forward NTT, short-distance levels by shuffles --------------------------------------
// r[i] = coefficient lane + 32 i throughout (in-place Cooley-Tukey order, ntt.hpp:74-86)
__device__ __forceinline__ void ntt_fwd_shfl(int32_t (&r)[8], const int2* zs, int lane) {
#pragma unroll
  for (int i = 0; i < 4; ++i) ct_bfly(r[i], r[i + 4], c_zeta[1]);
  ct_bfly(r[0], r[2], c_zeta[2]);
  ct_bfly(r[1], r[3], c_zeta[2]);
  ct_bfly(r[4], r[6], c_zeta[3]);
  ct_bfly(r[5], r[7], c_zeta[3]);
#pragma unroll
  for (int i = 0; i < 8; i += 2) ct_bfly(r[i], r[i + 1], c_zeta[4 + i / 2]);
#pragma unroll
  for (int len = 16; len >= 1; len >>= 1) {
    const bool upper = (lane & len) != 0;  // this lane holds the b operand of its butterflies
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int c = lane + 32 * i;
      const int2 z = zs[128 / len + c / (2 * len)];
      const int32_t p = __shfl_xor_sync(0xffffffffu, r[i], len);
      const int32_t bv = upper ? r[i] : p, av = upper ? p : r[i];
      const int32_t t = twiddle_mul(bv, z);
      r[i] = upper ? av - t : av + t;
    }
  }
}

__global__ void k_ntt(int32_t* polys, int reps, int variant) {
  __shared__ __align__(16) int2 zs[256], nzs[256];
  __shared__ __align__(16) int32_t tiles[4][kTileWords];
  load_twiddles(zs, nzs);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t w = blockIdx.x * 4 + warp;
  int32_t* a = polys + w * kN;
  int32_t r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) r[i] = a[lane + 32 * i];
  if (variant == 0) {
#pragma unroll 1
    for (int k = 0; k < reps; ++k) {
      ntt_fwd(r, tiles[warp], zs, lane);
      if (k + 1 < reps) {  // chain: feed the output back as the next input layout, reduced
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = reduce32(r[i]);
      }
    }
#pragma unroll
    for (int m = 0; m < 8; ++m) a[8 * lane + m] = freeze(r[m]);
  } else {
#pragma unroll 1
    for (int k = 0; k < reps; ++k) {
      ntt_fwd_shfl(r, zs, lane);
      if (k + 1 < reps) {
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = reduce32(r[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) a[lane + 32 * i] = freeze(r[i]);
  }
}

static float time_ms(void (*launch)(void*), void* ctx) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch(ctx);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    launch(ctx);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // ---- Keccak: correctness on 64 states, one permutation
  {
    const int n = 64;
    std::vector<uint64_t> h(n * 25), a(n * 25), b(n * 25);
    for (size_t i = 0; i < h.size(); ++i) h[i] = 0x9E3779B97F4A7C15ull * (i + 1) ^ (i << 17);
    uint64_t *d0, *d1;
    cudaMalloc(&d0, h.size() * 8);
    cudaMalloc(&d1, h.size() * 8);
    cudaMemcpy(d0, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(d1, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    k_keccak_thread<<<1, n>>>(d0, 3);
    k_keccak_coop<<<n / 4, 128>>>(d1, 3);
    cudaMemcpy(a.data(), d0, a.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), d1, b.size() * 8, cudaMemcpyDeviceToHost);
    printf("keccak: warp-cooperative == per-thread on %d states x 3 permutations: %s\n", n, a == b ? "yes" : "NO");
    cudaFree(d0);
    cudaFree(d1);
  }
  {
    const int perms = 200;
    const size_t n_thread = (size_t)sms * 16 * 128;  // 16 warps per SM, one state per thread
    const size_t n_coop = (size_t)sms * 16 * 4;      // 64 warps per SM (full occupancy), one state per warp
    uint64_t *d0, *d1;
    cudaMalloc(&d0, n_thread * 200);
    cudaMalloc(&d1, n_coop * 200);
    cudaMemset(d0, 1, n_thread * 200);
    cudaMemset(d1, 1, n_coop * 200);
    struct A { uint64_t* d; size_t n; int perms; } a0{d0, n_thread, perms}, a1{d1, n_coop, perms};
    const float t0 = time_ms([](void* p) { A* a = (A*)p; k_keccak_thread<<<a->n / 128, 128>>>(a->d, a->perms); }, &a0);
    const float t1 = time_ms([](void* p) { A* a = (A*)p; k_keccak_coop<<<a->n * 32 / 128, 128>>>(a->d, a->perms); }, &a1);
    const double r0 = n_thread * (double)perms / (t0 * 1e-3) / 1e9, r1 = n_coop * (double)perms / (t1 * 1e-3) / 1e9;
    printf("keccak: one state per thread  %.2f G permutations/s (16 warps/SM)\n", r0);
    printf("keccak: one state per 25 lanes %.2f G permutations/s (64 warps/SM)  -> per-thread mapping is %.1fx faster\n", r1, r0 / r1);
    cudaFree(d0);
    cudaFree(d1);
  }
  // ---- NTT
  {
    const size_t n = (size_t)sms * 64;
    std::vector<int32_t> h(n * kN), a(n * kN), b(n * kN);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (int32_t)((i * 2654435761u) % (uint32_t)kQ);
    int32_t *d0, *d1;
    cudaMalloc(&d0, h.size() * 4);
    cudaMalloc(&d1, h.size() * 4);
    cudaMemcpy(d0, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d1, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    k_ntt<<<n / 4, 128>>>(d0, 1, 0);
    k_ntt<<<n / 4, 128>>>(d1, 1, 1);
    cudaMemcpy(a.data(), d0, a.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(b.data(), d1, b.size() * 4, cudaMemcpyDeviceToHost);
    printf("ntt: shuffle variant == shared-memory-transpose variant on %zu polynomials: %s\n", n, a == b ? "yes" : "NO");
    struct A { int32_t* d; size_t n; int variant; } a0{d0, n, 0}, a1{d1, n, 1};
    const int reps = 400;
    static int s_reps = reps;
    const float t0 = time_ms([](void* p) { A* a = (A*)p; k_ntt<<<a->n / 4, 128>>>(a->d, s_reps, a->variant); }, &a0);
    const float t1 = time_ms([](void* p) { A* a = (A*)p; k_ntt<<<a->n / 4, 128>>>(a->d, s_reps, a->variant); }, &a1);
    const double r0 = n * (double)reps / (t0 * 1e-3) / 1e9, r1 = n * (double)reps / (t1 * 1e-3) / 1e9;
    printf("ntt: register passes + 2 shared-memory transposes %.3f G transforms/s\n", r0);
    printf("ntt: five levels by warp shuffles               %.3f G transforms/s  -> transposes are %.2fx faster\n", r1, r0 / r1);
  }
  return 0;
}
