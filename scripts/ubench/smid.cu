// Which SM does block b of a 4-CTAs-per-SM persistent grid land on?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(128, 4) k(unsigned* out, long long spin) {
  extern __shared__ unsigned char sm[];
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) out[blockIdx.x] = smid;
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
  if (spin < 0) sm[threadIdx.x] = 1;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 4;
  unsigned* d; cudaMalloc(&d, grid * 4);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 48000);
  k<<<grid, 128, 48000>>>(d, 2000000);
  unsigned* h = new unsigned[grid];
  cudaMemcpy(h, d, grid * 4, cudaMemcpyDeviceToHost);
  printf("sms %d\n", sms);
  for (int b = 0; b < 16; ++b) printf("block %d -> sm %u\n", b, h[b]);
  for (int b : {148, 149, 150, 296, 297, 444, 445, 591}) printf("block %d -> sm %u\n", b, h[b]);
  // co-residency of b and b + sms*j
  int same = 0;
  for (int b = 0; b < sms; ++b) same += (h[b] == h[b + sms]) + (h[b] == h[b + 2 * sms]) + (h[b] == h[b + 3 * sms]);
  printf("blocks b, b+148j on the same SM: %d of %d\n", same, 3 * sms);
  int adj = 0;
  for (int b = 0; b + 1 < grid; b += 2) adj += h[b] == h[b + 1];
  printf("blocks 2i, 2i+1 on the same SM: %d of %d\n", adj, grid / 2);
  return 0;
}
