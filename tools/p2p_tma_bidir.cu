// p2p_tma_bidir.cu — microbenchmark: bidirectional NVLink ring bandwidth when
// the data moves through the bulk-copy (TMA) engine instead of LSU loads.
// Every GPU i at once copies 1 GiB between itself and GPU (i+1) % n:
//   pull: cp.async.bulk peer global -> smem (mbarrier complete_tx), then
//         cp.async.bulk smem -> local global
//   push: local global -> smem, smem -> peer global
// one elected thread per CTA drives an S-stage ring of T-byte tiles; grid,
// T and S are swept.  The LSU copy (tools/p2p_bidir.cu) saturates at
// ~660 GB/s per direction pulling and ~698 pushing; the copy engines at 770.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/p2p_tma_bidir tools/p2p_tma_bidir.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e = (x);                                                       \
    if (e != cudaSuccess) {                                                    \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

constexpr int kMaxStages = 16;

// tile k of this CTA = global tile blockIdx.x + k * gridDim.x
__global__ void __launch_bounds__(32) tma_copy(const char* __restrict__ src, char* __restrict__ dst, long bytes,
                                                int tile, int stages) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bars[kMaxStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const long ntiles = bytes / tile;
  const long mine = ntiles > blockIdx.x ? (ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  auto issue = [&](long k) {
    const int s = (int)(k % stages);
    const long off = (blockIdx.x + k * (long)gridDim.x) * tile;
    mbar_expect_tx(&bars[s], tile);
    bulk_g2s(smem + (size_t)s * tile, src + off, tile, &bars[s]);
  };
  for (long k = 0; k < mine && k < stages; ++k) issue(k);
  for (long k = 0; k < mine; ++k) {
    const int s = (int)(k % stages);
    mbar_wait(&bars[s], (uint32_t)((k / stages) & 1));
    const long off = (blockIdx.x + k * (long)gridDim.x) * tile;
    bulk_s2g(dst + off, smem + (size_t)s * tile, tile);
    bulk_commit();
    bulk_wait_read1();   // tile k-1's store has read its stage: refill it
    if (k >= 1 && k - 1 + stages < mine) issue(k - 1 + stages);
  }
  bulk_wait_all();
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("{\"error\":\"needs 2 GPUs\"}\n");
    return 0;
  }
  const size_t bytes = size_t(1) << 30;
  std::vector<char*> a(n), b(n);
  std::vector<cudaStream_t> s(n);
  for (int i = 0; i < n; ++i) {
    CK(cudaSetDevice(i));
    for (int j = 0; j < n; ++j)
      if (j != i) cudaDeviceEnablePeerAccess(j, 0);
    cudaGetLastError();
    CK(cudaMalloc(&a[i], bytes));
    CK(cudaMalloc(&b[i], bytes));
    CK(cudaMemset(a[i], 1, bytes));
    CK(cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking));
    CK(cudaFuncSetAttribute(tma_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  }
  auto sync_all = [&]() {
    for (int i = 0; i < n; ++i) {
      CK(cudaSetDevice(i));
      CK(cudaDeviceSynchronize());
    }
  };
  auto timed = [&](int parts, auto fn) {
    std::vector<cudaEvent_t> e0(parts), e1(parts);
    for (int i = 0; i < parts; ++i) {
      CK(cudaSetDevice(i));
      CK(cudaEventCreate(&e0[i]));
      CK(cudaEventCreate(&e1[i]));
    }
    for (int w = 0; w < 2; ++w)
      for (int i = 0; i < parts; ++i) { CK(cudaSetDevice(i)); fn(i); }
    sync_all();
    const int it = 5;
    for (int i = 0; i < parts; ++i) { CK(cudaSetDevice(i)); CK(cudaEventRecord(e0[i], s[i])); }
    for (int k = 0; k < it; ++k)
      for (int i = 0; i < parts; ++i) { CK(cudaSetDevice(i)); fn(i); }
    for (int i = 0; i < parts; ++i) { CK(cudaSetDevice(i)); CK(cudaEventRecord(e1[i], s[i])); }
    sync_all();
    float worst = 0.f;
    for (int i = 0; i < parts; ++i) {
      float ms;
      CK(cudaEventElapsedTime(&ms, e0[i], e1[i]));
      if (ms > worst) worst = ms;
      CK(cudaEventDestroy(e0[i]));
      CK(cudaEventDestroy(e1[i]));
    }
    return (double)bytes * it / (worst * 1e-3) / 1e9;
  };
  const int parts = n;
  struct Cfg { int grid, tile, stages; };
  const Cfg cfgs[] = {{148, 8192, 4},   {148, 16384, 4},  {148, 32768, 4},  {148, 16384, 8},
                      {148, 32768, 6},  {296, 16384, 4},  {296, 32768, 3},  {444, 16384, 4},
                      {592, 16384, 3},  {148, 65536, 3},  {74, 32768, 6},   {296, 8192, 8}};
  for (const Cfg& c : cfgs) {
    const size_t sm = (size_t)c.tile * c.stages;
    double pull = timed(parts, [&](int i) {
      tma_copy<<<c.grid, 32, sm, s[i]>>>(a[(i + 1) % parts], b[i], (long)bytes, c.tile, c.stages);
    });
    double push = timed(parts, [&](int i) {
      tma_copy<<<c.grid, 32, sm, s[i]>>>(a[i], b[(i + 1) % parts], (long)bytes, c.tile, c.stages);
    });
    double pull1 = timed(1, [&](int i) {
      tma_copy<<<c.grid, 32, sm, s[0]>>>(a[1], b[0], (long)bytes, c.tile, c.stages);
    });
    printf("{\"gpus\":%d,\"pattern\":\"ring, every GPU at once (bidirectional), TMA bulk copy\",\"grid\":%d,"
           "\"tile\":%d,\"stages\":%d,\"pull_GBps\":%.1f,\"push_GBps\":%.1f,\"pull_one_direction_GBps\":%.1f}\n",
           parts, c.grid, c.tile, c.stages, pull, push, pull1);
    fflush(stdout);
  }
  return 0;
}
