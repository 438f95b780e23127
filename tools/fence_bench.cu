// fence_bench.cu — microbenchmark: the cost of the synchronisation
// primitives a cross-GPU barrier is made of, on two NVLink peers.
//   fence_sys      __threadfence_system() (fence.sc.sys), one thread
//   fence_gpu      __threadfence()
//   st_release_sys st.release.sys to a flag in the PEER's memory
//   st_relaxed_sys st.relaxed.sys to the peer flag
//   fence.acq_rel.sys alone and followed by three relaxed peer stores (a barrier's release)
//   pingpong       GPU0 writes flag k on GPU1, GPU1 answers k on GPU0 (one
//                  thread each, acquire/release sys): half the round trip is
//                  the one-way signalling latency a barrier pays
// each alone and with a background kernel pulling 1 GiB over NVLink on both
// GPUs (the situation inside the collective rounds).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fence_bench tools/fence_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
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
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// out[0] = ns per op
__global__ void prim_kernel(int which, uint64_t* peer_flag, uint64_t* local, int iters, double* out) {
  if (threadIdx.x || blockIdx.x) return;
  const uint64_t t0 = gtimer();
  for (int i = 0; i < iters; ++i) {
    local[i & 63] = i;   // a pending local store, as in a barrier after work
    switch (which) {
      case 0: __threadfence_system(); break;
      case 1: __threadfence(); break;
      case 2: st_release_sys(peer_flag, i); break;
      case 3: st_relaxed_sys(peer_flag, i); break;
      case 4: asm volatile("fence.acq_rel.sys;" ::: "memory"); break;
      case 5:
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        st_relaxed_sys(peer_flag, i);
        st_relaxed_sys(peer_flag + 1, i);
        st_relaxed_sys(peer_flag + 2, i);
        break;
    }
  }
  out[0] = (double)(gtimer() - t0) / iters;
}

// role 0: ping k, wait pong k; role 1: wait ping k, pong k
__global__ void pingpong_kernel(int role, uint64_t* my_flag, uint64_t* peer_flag, int iters, uint64_t base,
                                double* out) {
  if (threadIdx.x || blockIdx.x) return;
  const uint64_t t0 = gtimer();
  for (int i = 1; i <= iters; ++i) {
    const uint64_t v = base + i;
    if (role == 0) {
      st_release_sys(peer_flag, v);
      while (ld_acquire_sys(my_flag) < v) {
      }
    } else {
      while (ld_acquire_sys(my_flag) < v) {
      }
      st_release_sys(peer_flag, v);
    }
  }
  out[0] = (double)(gtimer() - t0) / iters;
}

__global__ void bg_pull(const uint4* __restrict__ src, uint4* __restrict__ dst, long n16) {
  const long stride = (long)gridDim.x * blockDim.x;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) __stcg(dst + i, __ldcg(src + i));
}

int main() {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (n < 2) {
    printf("{\"error\":\"needs 2 GPUs\"}\n");
    return 0;
  }
  const size_t bytes = size_t(1) << 30;
  uint64_t* flags[2];
  uint64_t* local[2];
  double* out[2];
  char *a[2], *b[2];
  cudaStream_t s[2], bg[2];
  for (int i = 0; i < 2; ++i) {
    CK(cudaSetDevice(i));
    cudaDeviceEnablePeerAccess(1 - i, 0);
    cudaGetLastError();
    CK(cudaMalloc(&flags[i], 4096));
    CK(cudaMemset(flags[i], 0, 4096));
    CK(cudaMalloc(&local[i], 4096));
    CK(cudaMallocManaged(&out[i], 64));
    CK(cudaMalloc(&a[i], bytes));
    CK(cudaMalloc(&b[i], bytes));
    CK(cudaStreamCreateWithFlags(&s[i], cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&bg[i], cudaStreamNonBlocking));
  }
  const char* names[] = {"fence_sys", "fence_gpu", "st_release_sys_peer", "st_relaxed_sys_peer",
                         "fence_acq_rel_sys", "fence_acq_rel_sys_then_3_relaxed_peer_stores"};
  uint64_t base = 0;
  for (int load = 0; load < 2; ++load) {
    if (load)
      for (int i = 0; i < 2; ++i) {
        CK(cudaSetDevice(i));
        for (int r = 0; r < 3; ++r)
          bg_pull<<<120, 1024, 0, bg[i]>>>((const uint4*)a[1 - i], (uint4*)b[i], (long)(bytes / 16));
      }
    for (int w = 0; w < 6; ++w) {
      CK(cudaSetDevice(0));
      prim_kernel<<<1, 32, 0, s[0]>>>(w, flags[1] + 8, local[0], 2000, out[0]);
      CK(cudaStreamSynchronize(s[0]));
      printf("{\"op\":\"%s\",\"background_nvlink_pull\":%d,\"ns\":%.1f}\n", names[w], load, out[0][0]);
    }
    for (int i = 0; i < 2; ++i) {
      CK(cudaSetDevice(i));
      pingpong_kernel<<<1, 32, 0, s[i]>>>(i, flags[i], flags[1 - i], 2000, base, out[i]);
    }
    base += 2000;
    for (int i = 0; i < 2; ++i) {
      CK(cudaSetDevice(i));
      CK(cudaStreamSynchronize(s[i]));
    }
    printf("{\"op\":\"pingpong_round_trip\",\"background_nvlink_pull\":%d,\"ns\":%.1f}\n", load, out[0][0]);
    for (int i = 0; i < 2; ++i) {
      CK(cudaSetDevice(i));
      CK(cudaDeviceSynchronize());
    }
  }
  return 0;
}
