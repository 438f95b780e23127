// stream_bw.cu — HBM ceiling of the Adam access pattern on one B200:
// (a) 1-read/1-write float4 copy; (b) the fused-Adam pattern without the
// arithmetic (read bf16 g + fp32 w/m/v, write fp32 w/m/v + bf16 p: 28 B/elem);
// (c) (b) with the full IEEE Adam arithmetic.  Grid-stride, 8 elements/thread.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/stream_bw tools/stream_bw.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>

__global__ void copy_k(const float4* __restrict__ a, float4* __restrict__ b, long n4) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}

template <bool MATH>
__global__ void adam_pattern(const uint4* __restrict__ g, float4* w, float4* m, float4* v, uint4* p, long n8) {
  for (long u = blockIdx.x * (long)blockDim.x + threadIdx.x; u < n8; u += (long)gridDim.x * blockDim.x) {
    uint4 gv = __ldcs(g + u);
    float4 w0 = __ldcs(w + 2 * u), w1 = __ldcs(w + 2 * u + 1);
    float4 m0 = __ldcs(m + 2 * u), m1 = __ldcs(m + 2 * u + 1);
    float4 v0 = __ldcs(v + 2 * u), v1 = __ldcs(v + 2 * u + 1);
    float gg[8] = {__uint_as_float(gv.x << 16), __uint_as_float(gv.x & 0xffff0000u), __uint_as_float(gv.y << 16),
                   __uint_as_float(gv.y & 0xffff0000u), __uint_as_float(gv.z << 16), __uint_as_float(gv.z & 0xffff0000u),
                   __uint_as_float(gv.w << 16), __uint_as_float(gv.w & 0xffff0000u)};
    float ww[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
    float mm[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
    float vv[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      if (MATH) {
        float gr = gg[e];
        mm[e] = __fadd_rn(__fmul_rn(0.9f, mm[e]), __fmul_rn(0.1f, gr));
        vv[e] = __fadd_rn(__fmul_rn(0.95f, vv[e]), __fmul_rn(0.05f, __fmul_rn(gr, gr)));
        float d = __fadd_rn(__fdiv_rn(__fsqrt_rn(vv[e]), 0.2f), 1e-8f);
        ww[e] = __fsub_rn(ww[e], __fmul_rn(3e-4f, __fdiv_rn(mm[e], d)));
      } else {
        mm[e] += gg[e];
        vv[e] += gg[e];
        ww[e] += gg[e];
      }
    }
    __stcs(w + 2 * u, make_float4(ww[0], ww[1], ww[2], ww[3]));
    __stcs(w + 2 * u + 1, make_float4(ww[4], ww[5], ww[6], ww[7]));
    __stcs(m + 2 * u, make_float4(mm[0], mm[1], mm[2], mm[3]));
    __stcs(m + 2 * u + 1, make_float4(mm[4], mm[5], mm[6], mm[7]));
    __stcs(v + 2 * u, make_float4(vv[0], vv[1], vv[2], vv[3]));
    __stcs(v + 2 * u + 1, make_float4(vv[4], vv[5], vv[6], vv[7]));
    __nv_bfloat162 b[4];
    for (int e = 0; e < 4; ++e) b[e] = __floats2bfloat162_rn(ww[2 * e], ww[2 * e + 1]);
    p[u] = *reinterpret_cast<uint4*>(b);
  }
}

int main() {
  const long n = 1l << 29;   // 536M elements: 15 GB of Adam traffic
  void *g, *w, *m, *v, *p, *a, *b;
  cudaMalloc(&g, n * 2); cudaMalloc(&w, n * 4); cudaMalloc(&m, n * 4); cudaMalloc(&v, n * 4); cudaMalloc(&p, n * 2);
  cudaMalloc(&a, n * 4); cudaMalloc(&b, n * 4);
  cudaMemset(g, 0, n * 2); cudaMemset(w, 0, n * 4); cudaMemset(m, 0, n * 4); cudaMemset(v, 0, n * 4);
  cudaMemset(a, 0, n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  int grids[] = {148 * 4, 148 * 8, 148 * 16, 148 * 32};
  for (int gr : grids) {
    for (int it = 0; it < 2; ++it) copy_k<<<gr, 256>>>((float4*)a, (float4*)b, n / 4);
    cudaEventRecord(e0);
    for (int it = 0; it < 5; ++it) copy_k<<<gr, 256>>>((float4*)a, (float4*)b, n / 4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"kernel\":\"copy\",\"grid\":%d,\"GBps\":%.1f}\n", gr, 8.0 * n / (ms / 5) / 1e6);
    for (int math = 0; math < 2; ++math) {
      auto k = math ? adam_pattern<true> : adam_pattern<false>;
      for (int it = 0; it < 2; ++it) k<<<gr, 256>>>((uint4*)g, (float4*)w, (float4*)m, (float4*)v, (uint4*)p, n / 8);
      cudaEventRecord(e0);
      for (int it = 0; it < 5; ++it) k<<<gr, 256>>>((uint4*)g, (float4*)w, (float4*)m, (float4*)v, (uint4*)p, n / 8);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"kernel\":\"adam_pattern%s\",\"grid\":%d,\"GBps\":%.1f}\n", math ? "_math" : "", gr,
             28.0 * n / (ms / 5) / 1e6);
    }
  }
  return 0;
}
