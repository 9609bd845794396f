// Does a second stream's kernel start on SM resources freed by CTAs of a first, still
// running, full-occupancy kernel?  (What sits in front of it in its stream matters.)
#include <cstdio>
#include <cuda_runtime.h>
struct T { unsigned long long first_start, last_start, first_exit, last_exit; };
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void __launch_bounds__(128, 4) big(T* t, unsigned long long base_ns) {
  extern __shared__ unsigned char sm[];
  if (threadIdx.x == 0) { unsigned long long n = gt(); atomicMin(&t->first_start, n); atomicMax(&t->last_start, n); }
  // block b runs base * (1 + b / grid): staggered exits
  const unsigned long long dur = base_ns + base_ns * blockIdx.x / gridDim.x;
  const unsigned long long t0 = gt();
  while (gt() - t0 < dur) { if (base_ns == 1) sm[threadIdx.x] = 1; }
  if (threadIdx.x == 0) { unsigned long long n = gt(); atomicMin(&t->first_exit, n); atomicMax(&t->last_exit, n); }
}
__global__ void small_nosmem(int* p) { if (p && threadIdx.x == 9999) p[0] = 1; }
__global__ void small_smem(int* p) { __shared__ int s[7000]; s[threadIdx.x] = 1; if (p && threadIdx.x == 9999) p[0] = s[0]; }
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 4, smem = 48000;
  cudaFuncSetAttribute(big, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  T *d, h[2];
  cudaMalloc(&d, 2 * sizeof(T));
  int* scratch; cudaMalloc(&scratch, 1 << 20);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  const char* names[] = {"plain", "small kernel (no smem) first", "small kernel (28 KB smem) first", "memsetAsync first",
                         "pageable H2D memcpyAsync first", "cudaFuncSetAttribute before launch", "small kernels first, all with carveout = max shared"};
  for (int v = 0; v < 7; ++v) {
    T init = {~0ull, 0, ~0ull, 0};
    T two[2] = {init, init};
    cudaMemcpy(d, two, sizeof two, cudaMemcpyHostToDevice);
    cudaDeviceSynchronize();
    if (v == 6) {
      cudaFuncSetAttribute(big, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
      cudaFuncSetAttribute(small_nosmem, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
      cudaFuncSetAttribute(small_smem, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    }
    big<<<grid, 128, smem, s1>>>(d, 2000000ull);  // 2..4 ms
    if (v == 6) { small_nosmem<<<8, 128, 0, s2>>>(nullptr); small_smem<<<8, 128, 0, s2>>>(nullptr); }
    if (v == 1) small_nosmem<<<8, 128, 0, s2>>>(nullptr);
    if (v == 2) small_smem<<<8, 128, 0, s2>>>(nullptr);
    if (v == 3) cudaMemsetAsync(scratch, 0, 4096, s2);
    int hv = 7;
    if (v == 4) cudaMemcpyAsync(scratch, &hv, sizeof hv, cudaMemcpyHostToDevice, s2);
    if (v == 5) cudaFuncSetAttribute(big, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    big<<<grid, 128, smem, s2>>>(d + 1, 2000000ull);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    const unsigned long long t0 = h[0].first_start;
    printf("%-36s K1 exits %.2f..%.2f ms | K2 first start %.2f last start %.2f, last exit %.2f\n", names[v],
           (h[0].first_exit - t0) / 1e6, (h[0].last_exit - t0) / 1e6, (h[1].first_start - t0) / 1e6,
           (h[1].last_start - t0) / 1e6, (h[1].last_exit - t0) / 1e6);
  }
  return 0;
}
