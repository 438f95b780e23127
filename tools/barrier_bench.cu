// barrier_bench.cu — microbenchmark: the cross-GPU grid barrier of the
// collective rounds kernel in isolation (148 CTAs per GPU, every GPU's grid
// synchronising with its ring neighbours, no data), variants:
//   0 relay      last-arriving CTA: fence.acq_rel.sys, relaxed flag stores to
//                the peers, polls their flags, opens a local go word (the
//                library's scheme, kernels.cu grid_peer_barrier)
//   1 relay+pa   the same followed by fence.proxy.async (what the TMA rounds
//                kernel adds after each barrier)
//   2 direct     every CTA polls the peers' flags itself (no go word)
//   3 relay-gpu  as 0 with a gpu-scope fence before the flag stores
//   4 relay-nots as 0 without the globaltimer timeout checks in the spin loops
// Prints us per barrier.  Build:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/barrier_bench tools/barrier_bench.cu
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

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

struct Args {
  uint64_t* peer_slot[2];   // my flag slot in each neighbour's memory
  uint64_t* my_flags;       // [2]: written by the neighbours
  unsigned long long* arrive;
  unsigned long long* go;
  int iters, variant;
  double* out;
};

__global__ void barrier_loop(Args a) {
  const uint64_t t0 = gtimer();
  for (int it = 1; it <= a.iters; ++it) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const unsigned long long target = (unsigned long long)it * gridDim.x;
      const unsigned long long old = atomicAdd(a.arrive, 1ull);
      const uint64_t val = it;
      const bool ts = a.variant != 4;
      if (a.variant == 2) {
        if (old + 1 == target) {
          asm volatile("fence.acq_rel.sys;" ::: "memory");
          st_relaxed_sys(a.peer_slot[0], val);
          st_relaxed_sys(a.peer_slot[1], val);
        }
        for (int x = 0; x < 2; ++x)
          while (ld_acquire_sys(&a.my_flags[x]) < val) {
            if (gtimer() - t0 > 20000000000ull) break;
          }
        while (ld_acquire_gpu(a.arrive) < target) {
        }
      } else if (old + 1 == target) {
        if (a.variant == 3) __threadfence();
        else asm volatile("fence.acq_rel.sys;" ::: "memory");
        st_relaxed_sys(a.peer_slot[0], val);
        st_relaxed_sys(a.peer_slot[1], val);
        for (int x = 0; x < 2; ++x)
          while (ld_acquire_sys(&a.my_flags[x]) < val) {
            if (ts && gtimer() - t0 > 20000000000ull) break;
          }
        st_release_gpu(a.go, (unsigned long long)val);
      } else {
        while (ld_acquire_gpu(a.go) < (unsigned long long)val) {
          if (ts && gtimer() - t0 > 20000000000ull) break;
          __nanosleep(32);
        }
      }
      if (a.variant == 1) asm volatile("fence.proxy.async;" ::: "memory");
    }
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.out[0] = 1e-3 * (double)(gtimer() - t0) / a.iters;
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("{\"error\":\"needs 2 GPUs\"}\n");
    return 0;
  }
  std::vector<uint64_t*> flags(n);
  std::vector<unsigned long long*> ctr(n);
  std::vector<double*> out(n);
  std::vector<cudaStream_t> s(n);
  for (int i = 0; i < n; ++i) {
    CK(cudaSetDevice(i));
    for (int j = 0; j < n; ++j)
      if (j != i) cudaDeviceEnablePeerAccess(j, 0);
    cudaGetLastError();
    CK(cudaMalloc(&flags[i], 4096));
    CK(cudaMalloc(&ctr[i], 4096));
    CK(cudaMallocManaged(&out[i], 64));
    CK(cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking));
  }
  const char* names[] = {"relay", "relay+fence.proxy.async", "direct", "relay-gpu-fence", "relay-no-timeout"};
  const int iters = 2000;
  for (int v = 0; v < 5; ++v) {
    for (int i = 0; i < n; ++i) {
      CK(cudaSetDevice(i));
      CK(cudaMemset(flags[i], 0, 4096));
      CK(cudaMemset(ctr[i], 0, 4096));
      CK(cudaDeviceSynchronize());
    }
    for (int i = 0; i < n; ++i) {
      CK(cudaSetDevice(i));
      Args a{};
      const int prev = (i + n - 1) % n, next = (i + 1) % n;
      // my_flags[0] is written by prev, my_flags[1] by next
      a.peer_slot[0] = flags[next] + 0;   // I am next's predecessor
      a.peer_slot[1] = flags[prev] + 1;   // I am prev's successor
      a.my_flags = flags[i];
      a.arrive = ctr[i];
      a.go = ctr[i] + 8;
      a.iters = iters;
      a.variant = v;
      a.out = out[i];
      barrier_loop<<<148, 256, 0, s[i]>>>(a);
    }
    double worst = 0;
    for (int i = 0; i < n; ++i) {
      CK(cudaSetDevice(i));
      CK(cudaStreamSynchronize(s[i]));
      if (out[i][0] > worst) worst = out[i][0];
    }
    printf("{\"gpus\":%d,\"variant\":\"%s\",\"us_per_barrier\":%.2f}\n", n, names[v], worst);
    fflush(stdout);
  }
  return 0;
}
