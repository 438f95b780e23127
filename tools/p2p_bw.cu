// p2p_bw.cu — microbenchmark: NVLink push (remote st.global) vs pull (remote
// ld.global) copy bandwidth between GPU 0 and GPU 1 for several CTA counts,
// block sizes and unroll depths; cudaMemcpyPeerAsync as reference.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o p2p_bw tools/p2p_bw.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

template <int UNR>
__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, long n16) {
  const long stride = (long)gridDim.x * blockDim.x;
  for (long base = (long)blockIdx.x * blockDim.x + threadIdx.x; base < n16; base += stride * UNR) {
    uint4 v[UNR];
#pragma unroll
    for (int k = 0; k < UNR; ++k)
      if (base + k * stride < n16) v[k] = __ldcg(src + base + k * stride);
#pragma unroll
    for (int k = 0; k < UNR; ++k)
      if (base + k * stride < n16) __stcg(dst + base + k * stride, v[k]);
  }
}

// block-contiguous slices (the rounds kernel's partition)
template <int UNR>
__global__ void copy_kernel_slices(const uint4* __restrict__ src, uint4* __restrict__ dst, long n16) {
  const long per = (n16 + gridDim.x - 1) / gridDim.x;
  const long b0 = blockIdx.x * per, b1 = min(n16, b0 + per);
  const long stride = blockDim.x;
  for (long base = b0 + threadIdx.x; base < b1; base += stride * UNR) {
    uint4 v[UNR];
#pragma unroll
    for (int k = 0; k < UNR; ++k)
      if (base + k * stride < b1) v[k] = __ldcg(src + base + k * stride);
#pragma unroll
    for (int k = 0; k < UNR; ++k)
      if (base + k * stride < b1) __stcg(dst + base + k * stride, v[k]);
  }
}

typedef void (*KFn)(const uint4*, uint4*, long);

float run(KFn k, int grid, int block, const uint4* src, uint4* dst, long n16, cudaStream_t s) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k<<<grid, block, 0, s>>>(src, dst, n16);
  cudaEventRecord(a, s);
  const int it = 10;
  for (int i = 0; i < it; ++i) k<<<grid, block, 0, s>>>(src, dst, n16);
  cudaEventRecord(b, s);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / it;
}

int main() {
  const size_t bytes = 1ull << 30;
  const long n16 = bytes / 16;
  int ndev;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    printf("need 2 GPUs\n");
    return 0;
  }
  void *b0, *b1, *l0;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&b1, bytes));
  CK(cudaSetDevice(0));
  CK(cudaMalloc(&b0, bytes));
  CK(cudaMalloc(&l0, bytes));
  CK(cudaMemset(b0, 1, bytes));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  cudaStream_t s;
  CK(cudaStreamCreate(&s));
  // reference
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaMemcpyPeerAsync(b1, 1, b0, 0, bytes, s);
    cudaEventRecord(a, s);
    for (int i = 0; i < 10; ++i) cudaMemcpyPeerAsync(b1, 1, b0, 0, bytes, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("{\"mode\":\"memcpyPeer\",\"GBps\":%.1f}\n", bytes / (ms / 10) / 1e6);
  }
  struct V {
    const char* name;
    KFn fn;
  } vars[] = {{"u2", copy_kernel<2>}, {"u4", copy_kernel<4>}, {"u8", copy_kernel<8>},
              {"slice_u2", copy_kernel_slices<2>}, {"slice_u4", copy_kernel_slices<4>}};
  int grids[] = {32, 64, 148, 296};
  int blocks[] = {256, 512, 1024};
  for (auto& v : vars)
    for (int g : grids)
      for (int bl : blocks) {
        float push = run(v.fn, g, bl, (const uint4*)b0, (uint4*)b1, n16, s);   // local -> peer
        float pull = run(v.fn, g, bl, (const uint4*)b1, (uint4*)l0, n16, s);   // peer -> local
        float local = run(v.fn, g, bl, (const uint4*)b0, (uint4*)l0, n16, s);  // local copy
        printf("{\"var\":\"%s\",\"grid\":%d,\"block\":%d,\"push_GBps\":%.1f,\"pull_GBps\":%.1f,\"local_GBps\":%.1f}\n",
               v.name, g, bl, bytes / push / 1e6, bytes / pull / 1e6, 2 * bytes / local / 1e6);
      }
  return 0;
}
