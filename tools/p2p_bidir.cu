// p2p_bidir.cu — microbenchmark: NVLink bandwidth with traffic in BOTH
// directions at once (the ring collectives' situation: every GPU reads from its
// predecessor while its successor reads from it).  One process, all visible
// GPUs; GPU i pulls (remote ld.global) or pushes (remote st.global) 1 GiB
// from/to GPU (i+1) % n, all concurrently; also cudaMemcpyPeerAsync in both
// directions, and a 2-peer ingress case (GPU 0 pulls from 1 and 2 at once).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/p2p_bidir tools/p2p_bidir.cu
#include <cuda_runtime.h>

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

__global__ void copy_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst, long n16) {
  const long stride = (long)gridDim.x * blockDim.x;
  for (long base = (long)blockIdx.x * blockDim.x + threadIdx.x; base < n16; base += stride * 4) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (base + k * stride < n16) v[k] = __ldcg(src + base + k * stride);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (base + k * stride < n16) __stcg(dst + base + k * stride, v[k]);
  }
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("{\"error\":\"needs 2 GPUs\"}\n");
    return 0;
  }
  const size_t bytes = size_t(1) << 30;
  const long n16 = bytes / 16;
  std::vector<char*> a(n), b(n), c(n);
  std::vector<cudaStream_t> s(n);
  for (int i = 0; i < n; ++i) {
    CK(cudaSetDevice(i));
    for (int j = 0; j < n; ++j)
      if (j != i) cudaDeviceEnablePeerAccess(j, 0);
    cudaGetLastError();
    CK(cudaMalloc(&a[i], bytes));
    CK(cudaMalloc(&b[i], bytes));
    CK(cudaMalloc(&c[i], bytes));
    CK(cudaMemset(a[i], 1, bytes));
    CK(cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking));
  }
  auto sync_all = [&]() {
    for (int i = 0; i < n; ++i) {
      CK(cudaSetDevice(i));
      CK(cudaDeviceSynchronize());
    }
  };
  // time `fn(i)` launched on every participating GPU concurrently; GB/s per GPU
  auto timed = [&](int parts, auto fn) {
    std::vector<cudaEvent_t> e0(parts), e1(parts);
    for (int i = 0; i < parts; ++i) {
      CK(cudaSetDevice(i));
      CK(cudaEventCreate(&e0[i]));
      CK(cudaEventCreate(&e1[i]));
    }
    for (int w = 0; w < 2; ++w) {
      for (int i = 0; i < parts; ++i) { CK(cudaSetDevice(i)); fn(i); }
    }
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
    }
    return (double)bytes * it / (worst * 1e-3) / 1e9;
  };
  const int grid = 148, block = 1024;
  for (int parts : {2, n}) {
    if (parts > n) continue;
    double pull = timed(parts, [&](int i) {
      copy_kernel<<<grid, block, 0, s[i]>>>((const uint4*)a[(i + 1) % parts], (uint4*)b[i], n16);
    });
    double push = timed(parts, [&](int i) {
      copy_kernel<<<grid, block, 0, s[i]>>>((const uint4*)a[i], (uint4*)b[(i + 1) % parts], n16);
    });
    double dma = timed(parts, [&](int i) {
      CK(cudaMemcpyPeerAsync(b[i], i, a[(i + 1) % parts], (i + 1) % parts, bytes, s[i]));
    });
    printf("{\"gpus\":%d,\"pattern\":\"ring, every GPU at once (bidirectional)\",\"pull_GBps\":%.1f,"
           "\"push_GBps\":%.1f,\"memcpyPeer_GBps\":%.1f}\n", parts, pull, push, dma);
  }
  {  // one direction only, for reference
    double pull1 = timed(1, [&](int i) {
      copy_kernel<<<grid, block, 0, s[0]>>>((const uint4*)a[1], (uint4*)b[0], n16);
    });
    printf("{\"gpus\":2,\"pattern\":\"GPU0 pulls from GPU1 alone\",\"pull_GBps\":%.1f}\n", pull1);
  }
  if (n >= 3) {  // ingress from two peers at once: two kernels on GPU 0
    cudaStream_t s2;
    CK(cudaSetDevice(0));
    CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cudaEvent_t e0, e1, f1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreate(&f1));
    for (int w = 0; w < 3; ++w) {
      if (w == 2) CK(cudaEventRecord(e0, s[0]));
      CK(cudaStreamWaitEvent(s2, e0, 0));
      copy_kernel<<<grid / 2, block, 0, s[0]>>>((const uint4*)a[1], (uint4*)b[0], n16);
      copy_kernel<<<grid / 2, block, 0, s2>>>((const uint4*)a[2], (uint4*)c[0], n16);
    }
    CK(cudaEventRecord(f1, s2));
    CK(cudaStreamWaitEvent(s[0], f1, 0));
    CK(cudaEventRecord(e1, s[0]));
    CK(cudaDeviceSynchronize());
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("{\"gpus\":3,\"pattern\":\"GPU0 pulls from GPU1 and GPU2 at once\",\"ingress_GBps\":%.1f}\n",
           2.0 * bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
