// tma_peer_test.cu — does cp.async.bulk (global -> shared, mbarrier
// complete_tx) accept an NVLink peer address?  GPU 0 bulk-copies a buffer that
// lives on GPU 1 and checks the bytes; also reports the bandwidth of a
// persistent bulk-copy pull kernel.  Build:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/tma_peer_test tools/tma_peer_test.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstdint>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int TILE = 32768;   // bytes per stage
constexpr int STAGES = 4;

__global__ void bulk_pull(const char* __restrict__ src, char* __restrict__ dst, long nbytes) {
  extern __shared__ __align__(128) char sm[];
  __shared__ uint64_t bar[STAGES];
  const long ntiles = nbytes / TILE;
  const long mine = (ntiles > blockIdx.x) ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](long k) {
    const int s = k % STAGES;
    const long t = blockIdx.x + k * gridDim.x;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(TILE) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(sm + s * TILE)),
                 "l"(src + t * TILE), "r"(TILE), "r"(su32(&bar[s]))
                 : "memory");
  };
  if (threadIdx.x == 0)
    for (long k = 0; k < STAGES && k < mine; ++k) issue(k);
  for (long k = 0; k < mine; ++k) {
    const int s = k % STAGES;
    const uint32_t ph = (k / STAGES) & 1;
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}" ::"r"(
            su32(&bar[s])),
        "r"(ph)
        : "memory");
    const long t = blockIdx.x + k * gridDim.x;
    const uint4* from = reinterpret_cast<const uint4*>(sm + s * TILE);
    uint4* to = reinterpret_cast<uint4*>(dst + t * TILE);
    for (int i = threadIdx.x; i < TILE / 16; i += blockDim.x) to[i] = from[i];
    __syncthreads();
    if (threadIdx.x == 0 && k + STAGES < mine) issue(k + STAGES);
  }
}

int main() {
  int n;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("{\"skip\":\"need 2 GPUs\"}\n");
    return 0;
  }
  const long bytes = 1l << 30;
  char *peer, *loc;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&peer, bytes));
  char* h = (char*)malloc(bytes);
  for (long i = 0; i < bytes; ++i) h[i] = (char)(i * 131 + 7);
  CK(cudaMemcpy(peer, h, bytes, cudaMemcpyHostToDevice));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&loc, bytes));
  CK(cudaFuncSetAttribute(bulk_pull, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE * STAGES));
  bulk_pull<<<148, 512, TILE * STAGES>>>(peer, loc, bytes);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  char* back = (char*)malloc(bytes);
  CK(cudaMemcpy(back, loc, bytes, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (long i = 0; i < bytes; ++i) bad += back[i] != h[i];
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) bulk_pull<<<148, 512, TILE * STAGES>>>(peer, loc, bytes);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("{\"bulk_pull_from_peer\":\"%s\",\"mismatches\":%ld,\"GBps\":%.1f}\n", bad ? "WRONG" : "ok", bad,
         bytes / (ms / 10) / 1e6);
  return 0;
}
