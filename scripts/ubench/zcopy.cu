// Zero-copy (kernel stores into pinned host memory) write bandwidth by store pattern:
// what the sign kernel's commit step can expect from PCIe.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

// A: one warp per 2420-byte row, 32-bit stores, 128 contiguous bytes per warp instruction
__global__ void k_rows32(const uint32_t* __restrict__ src, uint32_t* dst, int rows, int words) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = warp; r < rows; r += nw)
    for (int w = lane; w < words; w += 32) dst[(size_t)r * words + w] = src[(size_t)(r & 1023) * words + w];
}
// B: flat, 16-byte stores, 512 contiguous aligned bytes per warp instruction
__global__ void k_flat128(const uint4* __restrict__ src, uint4* dst, size_t n16) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) dst[i] = src[i & 0xFFFFF];
}
// C: flat, 32-bit stores, aligned
__global__ void k_flat32(const uint32_t* __restrict__ src, uint32_t* dst, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = src[i & 0xFFFFF];
}
// D: one warp per row, 16-byte stores after aligning the destination (head bytes word-wise)
__global__ void k_rows128(const uint32_t* __restrict__ src, uint32_t* dst, int rows, int words) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = warp; r < rows; r += nw) {
    uint32_t* d = dst + (size_t)r * words;
    const uint32_t* s = src + (size_t)(r & 1023) * words;
    const int head = (int)((16 - ((uintptr_t)d & 15)) & 15) >> 2;  // words until 16-byte alignment
    if (lane < head) d[lane] = s[lane];
    const int n16 = (words - head) / 4;
    uint4* d16 = reinterpret_cast<uint4*>(d + head);
    for (int c = lane; c < n16; c += 32) {
      const uint32_t* p = s + head + 4 * c;
      d16[c] = make_uint4(p[0], p[1], p[2], p[3]);
    }
    const int done = head + 4 * n16;
    if (lane < words - done) d[done + lane] = s[done + lane];
  }
}

int main() {
  const size_t bytes = 242000000;  // 100k signatures of 2420 bytes
  const int words = 605, rows = 100000;
  uint32_t *src, *host;
  cudaMalloc(&src, 16 << 20);
  cudaMemset(src, 7, 16 << 20);
  cudaHostAlloc(&host, bytes + 64, cudaHostAllocDefault);
  uint32_t* hd;
  cudaHostGetDevicePointer(&hd, host, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int grid : {148, 592, 2368}) {
    for (int v = 0; v < 4; ++v) {
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        if (v == 0) k_rows32<<<grid, 128>>>(src, hd, rows, words);
        if (v == 1) k_flat128<<<grid, 128>>>((const uint4*)src, (uint4*)hd, bytes / 16);
        if (v == 2) k_flat32<<<grid, 128>>>(src, hd, bytes / 4);
        if (v == 3) k_rows128<<<grid, 128>>>(src, hd, rows, words);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      const char* names[] = {"rows of 2420 B, 32-bit stores", "flat, 128-bit stores", "flat, 32-bit stores", "rows of 2420 B, 128-bit stores"};
      printf("grid %4d  %-32s %.2f ms  %.1f GB/s\n", grid, names[v], best, bytes / best / 1e6);
    }
  }
  // reference: the copy engine
  uint32_t* dbig; cudaMalloc(&dbig, bytes);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0); cudaMemcpyAsync(host, dbig, bytes, cudaMemcpyDeviceToHost); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf("cudaMemcpyAsync D2H (copy engine)            %.2f ms  %.1f GB/s\n", best, bytes / best / 1e6);
  return 0;
}
