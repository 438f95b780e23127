// kernels.cu — sm_100a kernels of the PaRO sync + update step.
//
// Nothing here is a dense contraction, so there are no tensor-core paths:
// every kernel is HBM- or NVLink-bound streaming code.
//  * rounds_kernel: fold tasks of a collective round; 128-bit coalesced loads
//    (ld.global.cg: L1 bypass, peers' lines are never cached stale), one
//    8-element unit per 16 B, grid barrier + release/acquire peer flags.
//  * adam_kernel: 28 B/elem single pass (ghat 2 + master/m/v 12 read,
//    master/m/v 12 + bf16 param 2 written), streaming cache hints, fp64 norm
//    partials through warp shuffles.
// Numerics follow DESIGN R2 / R5-R7: every fp32 op is an explicit _rn
// intrinsic, so nvcc cannot contract them to FMA; bf16 rounding is cvt.rn.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.h"

namespace paro {

namespace {

constexpr int kRoundsBlock = 512;
constexpr int kAdamBlock = 256;
constexpr uint64_t kTimeoutNs = 20ull * 1000 * 1000 * 1000;  // 20 s per wait

// ------------------------------------------------------------- bf16 helpers
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ uint32_t pack2_rn(float lo, float hi) {
  __nv_bfloat162 r = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&r);
}

__device__ __forceinline__ void unpack8(const uint4& v, float f[8]) {
  f[0] = bf_lo(v.x); f[1] = bf_hi(v.x); f[2] = bf_lo(v.y); f[3] = bf_hi(v.y);
  f[4] = bf_lo(v.z); f[5] = bf_hi(v.z); f[6] = bf_lo(v.w); f[7] = bf_hi(v.w);
}

__device__ __forceinline__ uint4 pack8(const float f[8]) {
  uint4 v;
  v.x = pack2_rn(f[0], f[1]); v.y = pack2_rn(f[2], f[3]);
  v.z = pack2_rn(f[4], f[5]); v.w = pack2_rn(f[6], f[7]);
  return v;
}

// x <- RNE_bf16(fp32(x) * alpha)  (pack / pre-divide, R4)
__device__ __forceinline__ void scale_round8(float f[8], float alpha) {
  float t[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) t[e] = __fmul_rn(f[e], alpha);
  uint4 p = pack8(t);
  unpack8(p, f);
}

// acc <- RNE_bf16(fp32(acc) + fp32(x))  (one hop, R2)
__device__ __forceinline__ void hop8(float acc[8], const float x[8]) {
  float t[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) t[e] = __fadd_rn(acc[e], x[e]);
  uint4 p = pack8(t);
  unpack8(p, acc);
}

// fp32 wire (reading A3): x <- fp32(x) * alpha, acc <- acc + x, no bf16 rounding
__device__ __forceinline__ void mul8(float f[8], float alpha) {
#pragma unroll
  for (int e = 0; e < 8; ++e) f[e] = __fmul_rn(f[e], alpha);
}
__device__ __forceinline__ void add8(float acc[8], const float x[8]) {
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = __fadd_rn(acc[e], x[e]);
}
// a raw gradient's pre-scaling and one hop, on the wire of the task / segment
__device__ __forceinline__ void pre8(float f[8], float alpha, bool wide) {
  if (wide) mul8(f, alpha);
  else scale_round8(f, alpha);
}
__device__ __forceinline__ void hopw8(float acc[8], const float x[8], bool wide) {
  if (wide) add8(acc, x);
  else hop8(acc, x);
}
__device__ __forceinline__ void f4x2(const float4& a, const float4& b, float f[8]) {
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

// ------------------------------------------------------------- sync helpers
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
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Grid-wide barrier of this rank, then release/acquire flags with `peers`.
// The last CTA of this GPU to arrive publishes to the peers, waits for their
// flags and opens the local `go` word; every other CTA waits on `go` only, so
// the sys-scope traffic is one writer and one poller per GPU.  Per-CTA fences
// are gpu-scope unless the launch stores into peer memory (push transport):
// pull launches write only local memory, and the releasing CTA's
// fence.acq_rel.sys + flag stores (a release pattern) is cumulative over what
// it acquired through the arrive counter (PTX memory model: causality order is
// transitive across the gpu-scope and sys-scope synchronisations).  Measured:
// 1 MiB all-reduce at 2 GPUs 44 -> 37 us, 1 GiB unchanged (profiles/r01).
// Returns false (and leaves a sticky error word) on timeout.
__device__ bool grid_peer_barrier(const RoundsArgs& a, uint64_t peers, int bidx, int narr, uint64_t gen0) {
  __shared__ int s_ok;
  __syncthreads();
  if (threadIdx.x == 0) {
    int ok = 1;
    volatile int* err = a.bar.err;
    if (a.sys_fence_all) __threadfence_system();   // remote NVLink stores visible system-wide
    else __threadfence();
    const unsigned long long target = (unsigned long long)(narr + 1) * gridDim.x;
    const unsigned long long old = atomicAdd(a.bar.arrive, 1ull);
    const uint64_t val = gen0 * 256ull + (uint64_t)bidx + 1ull;
    const uint64_t t0 = globaltimer();
    if (old + 1 == target) {          // last CTA of this GPU: publish to peers, wait for them
      // release pattern: one fence.acq_rel.sys, then relaxed sys-scope flag stores
      // (st.release.sys would fence again per peer: 1.7 us each, tools/fence_bench.cu)
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      for (int x = 0; x < 64; ++x)
        if ((peers >> x) & 1ull) st_relaxed_sys(a.bar.peer_slot[x], val);
      for (int x = 0; x < 64 && ok; ++x) {
        if (!((peers >> x) & 1ull)) continue;
        while (ld_acquire_sys(&a.bar.my_flags[x]) < val) {
          if (*err || globaltimer() - t0 > kTimeoutNs) { ok = 0; atomicExch((int*)err, 2); break; }
        }
      }
      st_release_gpu(a.bar.go, (unsigned long long)val);
    } else {
      while (ld_acquire_gpu(a.bar.go) < (unsigned long long)val) {
        if (*err || globaltimer() - t0 > kTimeoutNs) { ok = 0; atomicExch((int*)err, 2); break; }
        __nanosleep(32);
      }
    }
    if (*err) ok = 0;
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}

// The first barrier of a launch, before any of its work: every write it must
// publish was made by earlier kernels (stream-ordered before this one), so no
// grid arrival is needed: CTA 0 publishes to the peers (fence.acq_rel.sys, then
// relaxed flag stores), waits for their flags and opens `go` for the others.
// Removes the arrival of every CTA (and their launch skew) from the critical
// path of latency-bound launches.
__device__ bool entry_barrier(const RoundsArgs& a, uint64_t peers, int bidx, uint64_t gen0) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) {
    int ok = 1;
    volatile int* err = a.bar.err;
    const uint64_t val = gen0 * 256ull + (uint64_t)bidx + 1ull;
    const uint64_t t0 = globaltimer();
    if (blockIdx.x == 0) {
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      for (int x = 0; x < 64; ++x)
        if ((peers >> x) & 1ull) st_relaxed_sys(a.bar.peer_slot[x], val);
      for (int x = 0; x < 64 && ok; ++x) {
        if (!((peers >> x) & 1ull)) continue;
        while (ld_acquire_sys(&a.bar.my_flags[x]) < val) {
          if (*err || globaltimer() - t0 > kTimeoutNs) { ok = 0; atomicExch((int*)err, 2); break; }
        }
      }
      st_release_gpu(a.bar.go, (unsigned long long)val);
    } else {
      while (ld_acquire_gpu(a.bar.go) < (unsigned long long)val) {
        if (*err || globaltimer() - t0 > kTimeoutNs) { ok = 0; atomicExch((int*)err, 2); break; }
        __nanosleep(32);
      }
    }
    if (*err) ok = 0;
    s_ok = ok;
  }
  __syncthreads();
  return s_ok != 0;
}

// barrier k of a launch (bidx counts every barrier, narr the grid arrivals);
// barrier values are gen0 * 256 + k + 1, gen0 = the channel's launch generation
__device__ __forceinline__ bool launch_barrier(const RoundsArgs& a, uint64_t peers, int& bidx, int& narr,
                                               uint64_t gen0) {
  const bool ok = (bidx == 0 && a.entry_fast) ? entry_barrier(a, peers, bidx, gen0)
                                              : grid_peer_barrier(a, peers, bidx, narr++, gen0);
  ++bidx;
  return ok;
}

// the channel's launch generation, read by every CTA at start: the previous
// launch on this channel (same stream) has exited, so the value is stable
__device__ __forceinline__ uint64_t launch_gen(const RoundsArgs& a) {
  return a.bar.gen ? *reinterpret_cast<volatile unsigned long long*>(a.bar.gen) : 0ull;
}

// the last CTA to exit resets the arrival counter and advances the generation
// (every CTA has read it and passed every barrier by then)
__device__ __forceinline__ void launch_exit(const RoundsArgs& a, uint64_t gen0) {
  if (!a.bar.my_flags || threadIdx.x != 0) return;
  __threadfence();
  if (atomicAdd(a.bar.exitc, 1u) + 1u == gridDim.x) {
    atomicExch(a.bar.arrive, 0ull);
    atomicExch(a.bar.exitc, 0u);
    atomicExch(a.bar.gen, (unsigned long long)(gen0 + 1));
  }
}

// NVLink bytes of one task / tile, split by link class: every peer input is
// pulled, a peer destination pushed (device-counted "moved" bytes, reported by
// paro_step_stats)
__device__ __forceinline__ void count_moved(const DTask* tk, int64_t ne, unsigned long long& mi,
                                            unsigned long long& me) {
  mi += (unsigned long long)ne * tk->mv_intra;   // per-element bytes precomputed from the peer masks
  me += (unsigned long long)ne * tk->mv_inter;
}
__device__ __forceinline__ void flush_moved(unsigned long long* moved, unsigned long long mi,
                                            unsigned long long me) {
  if (!moved) return;
  if (mi) atomicAdd(moved, mi);
  if (me) atomicAdd(moved + 1, me);
}

// ------------------------------------------------------------- fold tasks
// Each task is spread over the whole grid, grid-stride interleaved (every
// warp touches consecutive 16-byte units; measured on B200: interleaving beats
// per-CTA contiguous slices, tools/p2p_bw.cu), UNR independent 128-bit loads
// per input in flight per thread before any use.
template <int NIN, int UNR>
__device__ __forceinline__ void run_fold(const DTask* __restrict__ t, float alpha) {
  const uint4* in[NIN];
#pragma unroll
  for (int i = 0; i < NIN; ++i) in[i] = reinterpret_cast<const uint4*>(t->in[i]);
  uint4* dst = reinterpret_cast<uint4*>(t->dst);
  const uint32_t raw = t->rawmask;
  const int64_t n8 = t->n8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t ub = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; ub < n8; ub += stride * UNR) {
    uint4 v[UNR][NIN];
#pragma unroll
    for (int k = 0; k < UNR; ++k) {
      const int64_t u = ub + k * stride;
      if (u < n8) {
#pragma unroll
        for (int i = 0; i < NIN; ++i) v[k][i] = __ldcg(in[i] + u);
      }
    }
#pragma unroll
    for (int k = 0; k < UNR; ++k) {
      const int64_t u = ub + k * stride;
      if (u >= n8) break;
      if (NIN == 1 && !(raw & 1u)) {   // plain copy (all-gather hop): no unpack
        __stcg(dst + u, v[k][0]);
        continue;
      }
      float acc[8];
      unpack8(v[k][0], acc);
      if (raw & 1u) scale_round8(acc, alpha);
#pragma unroll
      for (int i = 1; i < NIN; ++i) {
        float x[8];
        unpack8(v[k][i], x);
        if ((raw >> i) & 1u) scale_round8(x, alpha);
        hop8(acc, x);
      }
      __stcg(dst + u, pack8(acc));
    }
  }
}

// Any input count, flat or nested (nest > 1: nblk blocks of nest inputs, each
// block folded in order, then the block results in order, then the rest), on
// either wire.  Used for tasks beyond the specialised paths (> 3-4 inputs, the
// one-shot topology's N-input folds, fp32-wire tasks).
__device__ __noinline__ void run_fold_generic(const DTask* __restrict__ t, float alpha) {
  const int nin = t->nin;
  const uint32_t raw = t->rawmask, f32 = t->f32mask;
  const bool wide = t->out_f32 != 0;
  const int nest = t->nest > 1 ? t->nest : nin, nblk = t->nest > 1 ? t->nblk : 1;
  const int64_t n8 = t->n8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  auto load = [&](int i, int64_t u, float f[8]) {
    if ((f32 >> i) & 1u) {
      const float4* p = reinterpret_cast<const float4*>(t->in[i]) + 2 * u;
      f4x2(__ldcg(p), __ldcg(p + 1), f);
    } else {
      unpack8(__ldcg(reinterpret_cast<const uint4*>(t->in[i]) + u), f);
      if ((raw >> i) & 1u) pre8(f, alpha, wide);
    }
  };
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n8; u += stride) {
    float acc[8];
    int i = 0;
    for (int b = 0; b < nblk; ++b) {
      float blk[8];
      load(i++, u, blk);
      for (int q = 1; q < nest; ++q) {
        float x[8];
        load(i++, u, x);
        hopw8(blk, x, wide);
      }
      if (b == 0) {
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = blk[e];
      } else {
        hopw8(acc, blk, wide);
      }
    }
    for (; i < nin; ++i) {
      float x[8];
      load(i, u, x);
      hopw8(acc, x, wide);
    }
    if (wide) {
      float4* d = reinterpret_cast<float4*>(t->dst) + 2 * u;
      __stcg(d, make_float4(acc[0], acc[1], acc[2], acc[3]));
      __stcg(d + 1, make_float4(acc[4], acc[5], acc[6], acc[7]));
    } else {
      __stcg(reinterpret_cast<uint4*>(t->dst) + u, pack8(acc));
    }
  }
}

__device__ __forceinline__ void run_task(const DTask* __restrict__ t, float alpha) {
  if (t->out_f32 || t->nest > 1) {
    run_fold_generic(t, alpha);
    return;
  }
  switch (t->nin) {
    case 1: run_fold<1, 2>(t, alpha); break;
    case 2: run_fold<2, 1>(t, alpha); break;
    case 3: run_fold<3, 1>(t, alpha); break;
    case 4: run_fold<4, 1>(t, alpha); break;
    default: run_fold_generic(t, alpha); break;
  }
}

__device__ __forceinline__ void trace_stamp(const RoundsArgs& a, int slot) {
  if (a.trace && threadIdx.x == 0 && slot < kTraceSlots)
    a.trace[(size_t)blockIdx.x * kTraceSlots + slot] = globaltimer();
}

__global__ void __maxnreg__(48) rounds_kernel(const RoundsArgs a) {
  if (a.bar.err && *(volatile int*)a.bar.err) return;   // sticky device error: do nothing
  int bidx = 0, narr = 0;
  unsigned long long mi = 0, me = 0;
  const uint64_t gen0 = launch_gen(a);
  trace_stamp(a, 0);
  for (int r = 0; r < a.nrounds; ++r) {
    const DRound rd = a.rounds[r];
    if (a.bar.my_flags && !launch_barrier(a, rd.peers_before, bidx, narr, gen0)) return;
    trace_stamp(a, 1 + 2 * r);
    for (int ti = rd.t0; ti < rd.t1; ++ti) {
      run_task(a.tasks + ti, a.alpha);
      if (blockIdx.x == 0 && threadIdx.x == 0) count_moved(a.tasks + ti, a.tasks[ti].n8 * 8, mi, me);
    }
    __syncthreads();
    trace_stamp(a, 2 + 2 * r);
  }
  if (a.bar.my_flags && a.final_barrier && !launch_barrier(a, a.final_peers, bidx, narr, gen0)) return;
  if (threadIdx.x == 0) flush_moved(a.moved, mi, me);
  launch_exit(a, gen0);
  trace_stamp(a, kTraceSlots - 1);
}

// ------------------------------------------------------------- Adam
struct AdamScal {
  float b1, omb1, b2, omb2, step_size, bc2s, eps, decay, s_g, alpha;
  int has_wd;
};

__device__ __forceinline__ float adam_elem(float g, float& w, float& m, float& v, const AdamScal& c,
                                           double& nsq, int& bad, bool in_norm) {
  const float gr = __fmul_rn(g, c.s_g);
  if (!isfinite(g)) bad = 1;
  if (in_norm) nsq += (double)gr * (double)gr;
  float ww = w;
  if (c.has_wd) ww = __fmul_rn(ww, c.decay);
  const float m2 = __fadd_rn(__fmul_rn(c.b1, m), __fmul_rn(c.omb1, gr));
  const float v2 = __fadd_rn(__fmul_rn(c.b2, v), __fmul_rn(c.omb2, __fmul_rn(gr, gr)));
  const float d = __fadd_rn(__fdiv_rn(__fsqrt_rn(v2), c.bc2s), c.eps);
  const float w2 = __fsub_rn(ww, __fmul_rn(c.step_size, __fdiv_rn(m2, d)));
  w = w2;
  m = m2;
  v = v2;
  return w2;
}

// g_hat input i of an Adam segment at 8-element unit u, as fp32 (bf16 widened, or
// fp32 on the fp32 wire); raw gradients pre-scaled on the segment's wire
__device__ __forceinline__ void ld_gin8(const AdamSeg& sg, int i, int64_t u, float alpha, float f[8]) {
  if ((sg.gf32 >> i) & 1u) {
    const float4* p = reinterpret_cast<const float4*>(sg.gin[i]) + 2 * u;
    f4x2(__ldcs(p), __ldcs(p + 1), f);
  } else {
    unpack8(__ldcs(reinterpret_cast<const uint4*>(sg.gin[i]) + u), f);
    if ((sg.graw >> i) & 1u) pre8(f, alpha, sg.gwide != 0);
  }
}

__device__ __forceinline__ void adam_unit(const AdamSeg& sg, int64_t u, const AdamScal& c, double& nsq,
                                          int& bad) {
  float g[8];
  const float4* mp = reinterpret_cast<const float4*>(sg.master) + 2 * u;
  const float4* m1p = reinterpret_cast<const float4*>(sg.m) + 2 * u;
  const float4* v1p = reinterpret_cast<const float4*>(sg.v) + 2 * u;
  float4 w0, w1, m0, m1, v0, v1;
  if (!sg.gwide) {
    uint4 gv[kAdamMaxIn];
#pragma unroll
    for (int i = 0; i < kAdamMaxIn; ++i)
      if (i < sg.gnin) gv[i] = __ldcs(reinterpret_cast<const uint4*>(sg.gin[i]) + u);
    w0 = __ldcs(mp), w1 = __ldcs(mp + 1);
    m0 = __ldcs(m1p), m1 = __ldcs(m1p + 1);
    v0 = __ldcs(v1p), v1 = __ldcs(v1p + 1);
    // g_hat: fused final hop(s) of the reduction, canonical order (R2)
    unpack8(gv[0], g);
    if (sg.graw & 1u) scale_round8(g, c.alpha);
#pragma unroll
    for (int i = 1; i < kAdamMaxIn; ++i) {
      if (i < sg.gnin) {
        float x[8];
        unpack8(gv[i], x);
        if ((sg.graw >> i) & 1u) scale_round8(x, c.alpha);
        hop8(g, x);
      }
    }
  } else {   // fp32 wire: fp32 inputs / fp32 hops, g_hat stays fp32
    w0 = __ldcs(mp), w1 = __ldcs(mp + 1);
    m0 = __ldcs(m1p), m1 = __ldcs(m1p + 1);
    v0 = __ldcs(v1p), v1 = __ldcs(v1p + 1);
    ld_gin8(sg, 0, u, c.alpha, g);
    for (int i = 1; i < sg.gnin; ++i) {
      float x[8];
      ld_gin8(sg, i, u, c.alpha, x);
      add8(g, x);
    }
  }
  float w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
  float m[8] = {m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, m1.w};
  float v[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
  const bool in_norm = sg.in_norm != 0;
#pragma unroll
  for (int e = 0; e < 8; ++e) adam_elem(g[e], w[e], m[e], v[e], c, nsq, bad, in_norm);
  __stcs(reinterpret_cast<float4*>(sg.master) + 2 * u, make_float4(w[0], w[1], w[2], w[3]));
  __stcs(reinterpret_cast<float4*>(sg.master) + 2 * u + 1, make_float4(w[4], w[5], w[6], w[7]));
  __stcs(reinterpret_cast<float4*>(sg.m) + 2 * u, make_float4(m[0], m[1], m[2], m[3]));
  __stcs(reinterpret_cast<float4*>(sg.m) + 2 * u + 1, make_float4(m[4], m[5], m[6], m[7]));
  __stcs(reinterpret_cast<float4*>(sg.v) + 2 * u, make_float4(v[0], v[1], v[2], v[3]));
  __stcs(reinterpret_cast<float4*>(sg.v) + 2 * u + 1, make_float4(v[4], v[5], v[6], v[7]));
  // the bf16 parameter goes straight into its all-gather / parameter slot, and
  // (fused all-gather) into the consumers' parameter buffers over NVLink
  const uint4 pk = pack8(w);
  reinterpret_cast<uint4*>(sg.param)[u] = pk;
  for (int i = 0; i < sg.npush; ++i) __stcg(reinterpret_cast<uint4*>(sg.push[i]) + u, pk);
}

// after a fused all-gather, make this thread's remote stores visible system-wide
// before the kernel ends (the step-end peer barrier then publishes them)
__device__ __forceinline__ void push_fence(const AdamArgs& a) {
  int any = 0;
  for (int i = 0; i < a.nseg; ++i) any |= a.seg[i].npush;
  if (any) __threadfence_system();
}

__device__ __forceinline__ float unscale_of(const AdamArgs& a) { return a.s_g_dev ? *a.s_g_dev : a.s_g; }

__global__ void __launch_bounds__(kAdamBlock, 3) adam_kernel(const AdamArgs a) {
  if (a.skip && *a.skip) return;   // two-phase step: non-finite gradients, update skipped
  const AdamScal c{a.b1, a.omb1, a.b2, a.omb2, a.step_size, a.bc2s, a.eps, a.decay, unscale_of(a), a.alpha,
                   a.has_wd};
  int64_t U = 0;
  for (int i = 0; i < a.nseg; ++i) U += a.seg[i].n8;
  const int64_t per = (U + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = min(U, (int64_t)blockIdx.x * per);
  const int64_t b1 = min(U, b0 + per);
  double nsq = 0.0;
  int bad = 0;
  int64_t base = 0;
  unsigned long long mi = 0, me = 0;
  for (int i = 0; i < a.nseg && base < b1; ++i) {
    const AdamSeg& sg = a.seg[i];
    const int64_t n8 = sg.n8;
    const int64_t s = max(b0, base) - base, e = min(b1, base + n8) - base;
    for (int64_t u = s + threadIdx.x; u < e; u += blockDim.x) adam_unit(sg, u, c, nsq, bad);
    if (threadIdx.x == 0 && e > s) {
      for (int k = 0; k < sg.gnin; ++k)
        if ((sg.gpeer >> k) & 1u) (((sg.ginter >> k) & 1u) ? me : mi) += (unsigned long long)(e - s) * 8 *
                                                                          (((sg.gf32 >> k) & 1u) ? 4 : 2);
      for (int k = 0; k < sg.npush; ++k) (((sg.pinter >> k) & 1u) ? me : mi) += (unsigned long long)(e - s) * 16;
    }
    base += n8;
  }
  push_fence(a);
  if (threadIdx.x == 0) flush_moved(a.moved, mi, me);
  // block reduction of the norm partial: warp shuffles, then one warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, o);
  __shared__ double s_part[kAdamBlock / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_part[wid] = nsq;
  const int any_bad = __syncthreads_or(bad);
  if (wid == 0) {
    double x = (lane < (int)(blockDim.x / 32)) ? s_part[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) {
      a.partials[blockIdx.x] = x;
      if (any_bad) atomicOr(a.nonfinite, 1);
    }
  }
}

// ------------------------------------------------------------- Adam, TMA pipeline
// Same arithmetic as adam_kernel, but the operand streams are moved by the
// bulk-copy engine (cp.async.bulk, the non-tensor TMA path) into a ring of
// shared-memory stages guarded by mbarriers: one thread keeps kStages-1 tiles
// (up to ~170 KB per SM) in flight while 16 warps compute on the current one,
// so memory-level parallelism no longer costs registers.  Persistent grid:
// one CTA per SM, tiles dealt round-robin.  Inputs must be local memory.

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
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

struct TileRef {
  int seg;
  int64_t start;   // element offset inside the segment
  int n;           // elements in this tile (multiple of 8)
};

template <int kTile>
__device__ __forceinline__ bool tile_of(const AdamArgs& a, int64_t t, TileRef& out) {
  for (int i = 0; i < a.nseg; ++i) {
    const int64_t n = a.seg[i].n8 * 8;
    const int64_t nt = (n + kTile - 1) / kTile;
    if (t < nt) {
      out.seg = i;
      out.start = t * kTile;
      out.n = (int)min((int64_t)kTile, n - out.start);
      return true;
    }
    t -= nt;
  }
  return false;
}

// kStore = false: results are stored by the threads (st.global.cs);
// kStore = true: results are written back into the stage in shared memory and
// leave through bulk copies too (master, m, v, the bf16 parameter and, for the
// fused all-gather, the peers' parameter buffers): the stage is refilled one
// iteration later, once its stores have read it (wait_group.read 1).
// kWide: the launch has fp32 g_hat inputs (the fp32 wire): 4-byte slots per
// input, fp32 pre-scaling and hops; the bf16 instantiation keeps the
// bf16-only arithmetic, constant slot sizes and fewer instructions.
template <bool kStore, int kThr, bool kWide>
__global__ void __launch_bounds__(kThr, 1) adam_tma_kernel(const AdamArgs a, int gnin_max, int stages) {
  constexpr int kTmaTile = kThr * 8;   // elements per tile (8 per thread)
  constexpr int kGsz = kWide ? 4 : 2;  // bytes per g_hat element in a stage slot
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full_bar[4];
  if (a.skip && *a.skip) return;   // two-phase step: non-finite gradients, update skipped
  const AdamScal c{a.b1, a.omb1, a.b2, a.omb2, a.step_size, a.bc2s, a.eps, a.decay, unscale_of(a), a.alpha,
                   a.has_wd};
  constexpr size_t g_bytes = (size_t)kTmaTile * kGsz, f_bytes = (size_t)kTmaTile * 4;
  const size_t stage_bytes = gnin_max * g_bytes + 3 * f_bytes;
  int64_t done = 0;   // elements of this CTA's tiles (thread 0; moved-byte count at the end)
  int64_t total = 0;
  for (int i = 0; i < a.nseg; ++i) total += (a.seg[i].n8 * 8 + kTmaTile - 1) / kTmaTile;
  const int64_t mine = (total > blockIdx.x) ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(&full_bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t k) {   // thread 0: load tile k of this CTA into stage k % stages
    TileRef tr;
    tile_of<kTmaTile>(a, blockIdx.x + k * gridDim.x, tr);
    const AdamSeg& sg = a.seg[tr.seg];
    const int s = (int)(k % stages);
    unsigned char* base = smem + s * stage_bytes;
    const uint32_t fb = (uint32_t)tr.n * 4;
    done += tr.n;
    if (kWide) {
      uint32_t tx = 3 * fb;
      for (int i = 0; i < sg.gnin; ++i) tx += (uint32_t)tr.n * (((sg.gf32 >> i) & 1u) ? 4 : 2);
      mbar_expect_tx(&full_bar[s], tx);
      for (int i = 0; i < sg.gnin; ++i) {
        const int es = ((sg.gf32 >> i) & 1u) ? 4 : 2;
        bulk_g2s(base + i * g_bytes, reinterpret_cast<const unsigned char*>(sg.gin[i]) + (size_t)tr.start * es,
                 (uint32_t)tr.n * es, &full_bar[s]);
      }
    } else {
      const uint32_t gb = (uint32_t)tr.n * 2;
      mbar_expect_tx(&full_bar[s], sg.gnin * gb + 3 * fb);
      for (int i = 0; i < sg.gnin; ++i) bulk_g2s(base + i * g_bytes, sg.gin[i] + tr.start, gb, &full_bar[s]);
    }
    unsigned char* fbase = base + gnin_max * g_bytes;
    bulk_g2s(fbase, sg.master + tr.start, fb, &full_bar[s]);
    bulk_g2s(fbase + f_bytes, sg.m + tr.start, fb, &full_bar[s]);
    bulk_g2s(fbase + 2 * f_bytes, sg.v + tr.start, fb, &full_bar[s]);
  };
  if (threadIdx.x == 0)
    for (int64_t k = 0; k < min((int64_t)stages, mine); ++k) issue(k);
  double nsq = 0.0;
  int bad = 0;
  for (int64_t k = 0; k < mine; ++k) {
    const int s = (int)(k % stages);
    mbar_wait(&full_bar[s], (uint32_t)((k / stages) & 1));
    TileRef tr;
    tile_of<kTmaTile>(a, blockIdx.x + k * gridDim.x, tr);
    const AdamSeg& sg = a.seg[tr.seg];
    unsigned char* base = smem + s * stage_bytes;
    const int e0 = threadIdx.x * 8;
    const bool act = e0 < tr.n;
    float* fw = reinterpret_cast<float*>(base + gnin_max * g_bytes);
    float w[8], m[8], v[8];
    uint4 pk = make_uint4(0, 0, 0, 0);
    if (act) {
      float g[8];
      if (kWide) {
        auto ld = [&](int i, float f[8]) {   // g_hat input i of this thread's 8 elements, from the stage
          if ((sg.gf32 >> i) & 1u) {
            const float4* q = reinterpret_cast<const float4*>(base + i * g_bytes + (size_t)e0 * 4);
            f4x2(q[0], q[1], f);
          } else {
            unpack8(*reinterpret_cast<const uint4*>(base + i * g_bytes + (size_t)e0 * 2), f);
            if ((sg.graw >> i) & 1u) mul8(f, c.alpha);
          }
        };
        ld(0, g);
        for (int i = 1; i < sg.gnin; ++i) {
          float x[8];
          ld(i, x);
          add8(g, x);
        }
      } else {
        unpack8(*reinterpret_cast<const uint4*>(base + e0 * 2), g);
        if (sg.graw & 1u) scale_round8(g, c.alpha);
        for (int i = 1; i < sg.gnin; ++i) {
          float x[8];
          unpack8(*reinterpret_cast<const uint4*>(base + i * g_bytes + e0 * 2), x);
          if ((sg.graw >> i) & 1u) scale_round8(x, c.alpha);
          hop8(g, x);
        }
      }
      const float4 w0 = *reinterpret_cast<const float4*>(fw + e0), w1 = *reinterpret_cast<const float4*>(fw + e0 + 4);
      const float4 m0 = *reinterpret_cast<const float4*>(fw + kTmaTile + e0);
      const float4 m1 = *reinterpret_cast<const float4*>(fw + kTmaTile + e0 + 4);
      const float4 v0 = *reinterpret_cast<const float4*>(fw + 2 * kTmaTile + e0);
      const float4 v1 = *reinterpret_cast<const float4*>(fw + 2 * kTmaTile + e0 + 4);
      f4x2(w0, w1, w);
      f4x2(m0, m1, m);
      f4x2(v0, v1, v);
      const bool in_norm = sg.in_norm != 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) adam_elem(g[e], w[e], m[e], v[e], c, nsq, bad, in_norm);
      pk = pack8(w);
    }
    if (kStore) {
      // fp32 inputs: every thread has read its input-0 bytes before the bf16
      // outputs (half their width) are written over them
      if (kWide) __syncthreads();
      if (act) {   // back into the stage, in place (each thread owns its 8 elements)
        *reinterpret_cast<float4*>(fw + e0) = make_float4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<float4*>(fw + e0 + 4) = make_float4(w[4], w[5], w[6], w[7]);
        *reinterpret_cast<float4*>(fw + kTmaTile + e0) = make_float4(m[0], m[1], m[2], m[3]);
        *reinterpret_cast<float4*>(fw + kTmaTile + e0 + 4) = make_float4(m[4], m[5], m[6], m[7]);
        *reinterpret_cast<float4*>(fw + 2 * kTmaTile + e0) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(fw + 2 * kTmaTile + e0 + 4) = make_float4(v[4], v[5], v[6], v[7]);
        *reinterpret_cast<uint4*>(base + e0 * 2) = pk;   // over g_hat input 0 (consumed)
      }
    } else if (act) {
      const int64_t o = tr.start + e0;
      __stcs(reinterpret_cast<float4*>(sg.master + o), make_float4(w[0], w[1], w[2], w[3]));
      __stcs(reinterpret_cast<float4*>(sg.master + o) + 1, make_float4(w[4], w[5], w[6], w[7]));
      __stcs(reinterpret_cast<float4*>(sg.m + o), make_float4(m[0], m[1], m[2], m[3]));
      __stcs(reinterpret_cast<float4*>(sg.m + o) + 1, make_float4(m[4], m[5], m[6], m[7]));
      __stcs(reinterpret_cast<float4*>(sg.v + o), make_float4(v[0], v[1], v[2], v[3]));
      __stcs(reinterpret_cast<float4*>(sg.v + o) + 1, make_float4(v[4], v[5], v[6], v[7]));
      *reinterpret_cast<uint4*>(sg.param + o) = pk;
      for (int i = 0; i < sg.npush; ++i) __stcg(reinterpret_cast<uint4*>(sg.push[i] + o), pk);
    }
    if (kStore) {
      fence_proxy_async_smem();   // this thread's smem writes -> visible to the bulk-copy engine
      __syncthreads();
      if (threadIdx.x == 0) {
        const uint32_t gb = (uint32_t)tr.n * 2, fb = (uint32_t)tr.n * 4;
        const unsigned char* fbase = base + gnin_max * g_bytes;
        bulk_s2g(sg.master + tr.start, fbase, fb);
        bulk_s2g(sg.m + tr.start, fbase + f_bytes, fb);
        bulk_s2g(sg.v + tr.start, fbase + 2 * f_bytes, fb);
        bulk_s2g(sg.param + tr.start, base, gb);
        for (int i = 0; i < sg.npush; ++i) bulk_s2g(sg.push[i] + tr.start, base, gb);
        bulk_commit();
        // the previous tile's stores have read their stage: refill it
        bulk_wait_read<1>();
        if (k >= 1 && k - 1 + stages < mine) issue(k - 1 + stages);
      }
    } else {
      __syncthreads();   // every thread is done with stage s: refill it
      if (threadIdx.x == 0 && k + stages < mine) issue(k + stages);
    }
  }
  if (kStore) {
    if (threadIdx.x == 0) {
      bulk_wait_all();
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __threadfence_system();
    }
  } else {
    push_fence(a);
  }
  if (threadIdx.x == 0 && a.moved && done > 0) {   // NVLink bytes of this CTA's tiles (real mode: one segment)
    const AdamSeg& sg = a.seg[0];
    unsigned long long mi = 0, me = 0;
    for (int i = 0; i < sg.gnin; ++i)
      if ((sg.gpeer >> i) & 1u)
        (((sg.ginter >> i) & 1u) ? me : mi) += (unsigned long long)done * (((sg.gf32 >> i) & 1u) ? 4 : 2);
    for (int i = 0; i < sg.npush; ++i) (((sg.pinter >> i) & 1u) ? me : mi) += (unsigned long long)done * 2;
    flush_moved(a.moved, mi, me);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, o);
  __shared__ double s_part[kThr / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_part[wid] = nsq;
  const int any_bad = __syncthreads_or(bad);
  if (wid == 0) {
    double x = (lane < (int)(blockDim.x / 32)) ? s_part[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) {
      a.partials[blockIdx.x] = x;
      if (any_bad) atomicOr(a.nonfinite, 1);
    }
  }
}

// ------------------------------------------------------------- Adam, warp-specialized TMA pipeline
// The TMA-store Adam with a dedicated producer warp: the kThr compute threads
// never wait for each other.  Per stage two mbarriers: `full` (the bulk loads
// landed) and `done` (every compute thread wrote its results back into the
// stage and fenced them for the async proxy).  The producer lane waits on
// `done`, sends the tile's results out with bulk stores, and refills the stage
// of the previous tile as soon as its stores have read it (wait_group.read 1).
// Same arithmetic, bits and bytes as adam_tma_kernel<true, kThr, kWide>.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int kThr, bool kWide>
__global__ void __launch_bounds__(kThr + 32, 1) adam_tma_ws_kernel(const AdamArgs a, int gnin_max, int stages) {
  constexpr int kTmaTile = kThr * 8;
  constexpr int kGsz = kWide ? 4 : 2;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full_bar[4], done_bar[4];
  if (a.skip && *a.skip) return;   // two-phase step: non-finite gradients, update skipped
  const AdamScal c{a.b1, a.omb1, a.b2, a.omb2, a.step_size, a.bc2s, a.eps, a.decay, unscale_of(a), a.alpha,
                   a.has_wd};
  constexpr size_t g_bytes = (size_t)kTmaTile * kGsz, f_bytes = (size_t)kTmaTile * 4;
  const size_t stage_bytes = gnin_max * g_bytes + 3 * f_bytes;
  int64_t total = 0;
  for (int i = 0; i < a.nseg; ++i) total += (a.seg[i].n8 * 8 + kTmaTile - 1) / kTmaTile;
  const int64_t mine = (total > blockIdx.x) ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const bool producer = threadIdx.x >= kThr;
  if (threadIdx.x == kThr) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&done_bar[s], kThr);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double nsq = 0.0;
  int bad = 0;
  if (producer) {
    if (threadIdx.x == kThr) {
      int64_t done = 0;
      auto issue = [&](int64_t k) {   // load tile k of this CTA into stage k % stages
        TileRef tr;
        tile_of<kTmaTile>(a, blockIdx.x + k * gridDim.x, tr);
        const AdamSeg& sg = a.seg[tr.seg];
        const int s = (int)(k % stages);
        unsigned char* base = smem + s * stage_bytes;
        const uint32_t fb = (uint32_t)tr.n * 4;
        done += tr.n;
        if (kWide) {
          uint32_t tx = 3 * fb;
          for (int i = 0; i < sg.gnin; ++i) tx += (uint32_t)tr.n * (((sg.gf32 >> i) & 1u) ? 4 : 2);
          mbar_expect_tx(&full_bar[s], tx);
          for (int i = 0; i < sg.gnin; ++i) {
            const int es = ((sg.gf32 >> i) & 1u) ? 4 : 2;
            bulk_g2s(base + i * g_bytes, reinterpret_cast<const unsigned char*>(sg.gin[i]) + (size_t)tr.start * es,
                     (uint32_t)tr.n * es, &full_bar[s]);
          }
        } else {
          const uint32_t gb = (uint32_t)tr.n * 2;
          mbar_expect_tx(&full_bar[s], sg.gnin * gb + 3 * fb);
          for (int i = 0; i < sg.gnin; ++i) bulk_g2s(base + i * g_bytes, sg.gin[i] + tr.start, gb, &full_bar[s]);
        }
        unsigned char* fbase = base + gnin_max * g_bytes;
        bulk_g2s(fbase, sg.master + tr.start, fb, &full_bar[s]);
        bulk_g2s(fbase + f_bytes, sg.m + tr.start, fb, &full_bar[s]);
        bulk_g2s(fbase + 2 * f_bytes, sg.v + tr.start, fb, &full_bar[s]);
      };
      for (int64_t k = 0; k < min((int64_t)stages, mine); ++k) issue(k);
      for (int64_t k = 0; k < mine; ++k) {
        const int s = (int)(k % stages);
        mbar_wait(&done_bar[s], (uint32_t)((k / stages) & 1));   // the compute threads' results are in
        TileRef tr;
        tile_of<kTmaTile>(a, blockIdx.x + k * gridDim.x, tr);
        const AdamSeg& sg = a.seg[tr.seg];
        unsigned char* base = smem + s * stage_bytes;
        const uint32_t gb = (uint32_t)tr.n * 2, fb = (uint32_t)tr.n * 4;
        const unsigned char* fbase = base + gnin_max * g_bytes;
        bulk_s2g(sg.master + tr.start, fbase, fb);
        bulk_s2g(sg.m + tr.start, fbase + f_bytes, fb);
        bulk_s2g(sg.v + tr.start, fbase + 2 * f_bytes, fb);
        bulk_s2g(sg.param + tr.start, base, gb);
        for (int i = 0; i < sg.npush; ++i) bulk_s2g(sg.push[i] + tr.start, base, gb);
        bulk_commit();
        bulk_wait_read<1>();   // the previous tile's stores have read their stage: refill it
        if (k >= 1 && k - 1 + stages < mine) issue(k - 1 + stages);
      }
      bulk_wait_all();
      asm volatile("fence.proxy.async.global;" ::: "memory");
      __threadfence_system();
      if (a.moved && done > 0) {   // NVLink bytes of this CTA's tiles (real mode: one segment)
        const AdamSeg& sg = a.seg[0];
        unsigned long long mi = 0, me = 0;
        for (int i = 0; i < sg.gnin; ++i)
          if ((sg.gpeer >> i) & 1u)
            (((sg.ginter >> i) & 1u) ? me : mi) += (unsigned long long)done * (((sg.gf32 >> i) & 1u) ? 4 : 2);
        for (int i = 0; i < sg.npush; ++i) (((sg.pinter >> i) & 1u) ? me : mi) += (unsigned long long)done * 2;
        flush_moved(a.moved, mi, me);
      }
    }
  } else {
    for (int64_t k = 0; k < mine; ++k) {
      const int s = (int)(k % stages);
      mbar_wait(&full_bar[s], (uint32_t)((k / stages) & 1));
      TileRef tr;
      tile_of<kTmaTile>(a, blockIdx.x + k * gridDim.x, tr);
      const AdamSeg& sg = a.seg[tr.seg];
      unsigned char* base = smem + s * stage_bytes;
      const int e0 = threadIdx.x * 8;
      const bool act = e0 < tr.n;
      float* fw = reinterpret_cast<float*>(base + gnin_max * g_bytes);
      float w[8], m[8], v[8];
      uint4 pk = make_uint4(0, 0, 0, 0);
      if (act) {
        float g[8];
        if (kWide) {
          auto ld = [&](int i, float f[8]) {
            if ((sg.gf32 >> i) & 1u) {
              const float4* q = reinterpret_cast<const float4*>(base + i * g_bytes + (size_t)e0 * 4);
              f4x2(q[0], q[1], f);
            } else {
              unpack8(*reinterpret_cast<const uint4*>(base + i * g_bytes + (size_t)e0 * 2), f);
              if ((sg.graw >> i) & 1u) mul8(f, c.alpha);
            }
          };
          ld(0, g);
          for (int i = 1; i < sg.gnin; ++i) {
            float x[8];
            ld(i, x);
            add8(g, x);
          }
        } else {
          unpack8(*reinterpret_cast<const uint4*>(base + e0 * 2), g);
          if (sg.graw & 1u) scale_round8(g, c.alpha);
          for (int i = 1; i < sg.gnin; ++i) {
            float x[8];
            unpack8(*reinterpret_cast<const uint4*>(base + i * g_bytes + e0 * 2), x);
            if ((sg.graw >> i) & 1u) scale_round8(x, c.alpha);
            hop8(g, x);
          }
        }
        const float4 w0 = *reinterpret_cast<const float4*>(fw + e0), w1 = *reinterpret_cast<const float4*>(fw + e0 + 4);
        const float4 m0 = *reinterpret_cast<const float4*>(fw + kTmaTile + e0);
        const float4 m1 = *reinterpret_cast<const float4*>(fw + kTmaTile + e0 + 4);
        const float4 v0 = *reinterpret_cast<const float4*>(fw + 2 * kTmaTile + e0);
        const float4 v1 = *reinterpret_cast<const float4*>(fw + 2 * kTmaTile + e0 + 4);
        f4x2(w0, w1, w);
        f4x2(m0, m1, m);
        f4x2(v0, v1, v);
        const bool in_norm = sg.in_norm != 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) adam_elem(g[e], w[e], m[e], v[e], c, nsq, bad, in_norm);
        pk = pack8(w);
      }
      // fp32 inputs: every compute thread has read its input-0 bytes before the
      // bf16 outputs are written over them (named barrier of the compute threads)
      if (kWide) asm volatile("bar.sync 1, %0;" ::"n"(kThr) : "memory");
      if (act) {
        *reinterpret_cast<float4*>(fw + e0) = make_float4(w[0], w[1], w[2], w[3]);
        *reinterpret_cast<float4*>(fw + e0 + 4) = make_float4(w[4], w[5], w[6], w[7]);
        *reinterpret_cast<float4*>(fw + kTmaTile + e0) = make_float4(m[0], m[1], m[2], m[3]);
        *reinterpret_cast<float4*>(fw + kTmaTile + e0 + 4) = make_float4(m[4], m[5], m[6], m[7]);
        *reinterpret_cast<float4*>(fw + 2 * kTmaTile + e0) = make_float4(v[0], v[1], v[2], v[3]);
        *reinterpret_cast<float4*>(fw + 2 * kTmaTile + e0 + 4) = make_float4(v[4], v[5], v[6], v[7]);
        *reinterpret_cast<uint4*>(base + e0 * 2) = pk;   // over g_hat input 0 (consumed)
      }
      fence_proxy_async_smem();   // this thread's smem writes -> visible to the bulk-copy engine
      mbar_arrive(&done_bar[s]);
    }
  }
  // norm partials (the producer warp contributes zeros)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, o);
  __shared__ double s_part[(kThr + 32) / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_part[wid] = nsq;
  const int any_bad = __syncthreads_or(bad);
  if (wid == 0) {
    double x = (lane < (int)(blockDim.x / 32)) ? s_part[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) {
      a.partials[blockIdx.x] = x;
      if (any_bad) atomicOr(a.nonfinite, 1);
    }
  }
}

// ------------------------------------------------------------- rounds, TMA pipeline
// The collective rounds with the operand streams moved by the bulk-copy engine:
// for every tile of a fold task, one thread issues cp.async.bulk for each input
// — NVLink-peer or local — into a 4-stage shared-memory ring (mbarrier
// complete_tx); 8 warps fold from shared memory and store the result.
// Memory-level parallelism no longer costs registers, so the kernel keeps
// NVLink busy beside the Adam kernel.  A stage holds one slot of `slotb` bytes
// per input: 8 KB (4096 bf16 / 2048 fp32 elements) for tasks of up to 3 inputs,
// smaller slots for the N-input folds of the one-shot topology (the stages
// stay within 96 KB).
constexpr int kRtThreads = 256;
constexpr int kRtSlotB = 8192;    // slot bytes per input for <= 3 inputs
constexpr int kRtStages = 4;      // stages for <= 3 inputs (8 KB slots)
constexpr int kRtMaxStages = 8;
constexpr int kRtMaxIn = kDevMaxIn;
constexpr int kRtSmem = kRtStages * 3 * kRtSlotB;   // 96 KB

// log2 of the slot bytes: 8 KB up to 4 inputs, else the largest power of two
// with 3 stages x max_in slots <= 96 KB (4 KB for 5-8 inputs, 2 KB for 9-16)
int rt_slot_lg(int max_in) {
  if (max_in <= 3) return 13;
  static const int env = std::getenv("PARO_RT_SLOT_LG") ? std::atoi(std::getenv("PARO_RT_SLOT_LG")) : 0;
  int lg = 13;   // the largest slot with >= 3 stages in 96 KB (larger bulk copies move more per request)
  while (lg > 10 && (3 * max_in) << lg > kRtSmem) --lg;
  if (env >= 10 && env <= 13 && (2 * max_in) << env <= kRtSmem) lg = env;
  return lg;
}
int rt_slot_bytes(int max_in) { return 1 << rt_slot_lg(max_in); }
// stages: 4 for <= 3 inputs (the tuned 8 KB-slot pipeline), else as many as
// fit the 96 KB (up to 8); PARO_RT_STAGES overrides both (A/B runs)
int rt_stages(int max_in) {
  static const int env = std::getenv("PARO_RT_STAGES") ? std::atoi(std::getenv("PARO_RT_STAGES")) : 0;
  int st = max_in <= 3 ? kRtStages : kRtSmem / (max_in << rt_slot_lg(max_in));
  if (env >= 2) st = std::min(env, kRtSmem / (max_in << rt_slot_lg(max_in)));
  return std::max(2, std::min(kRtMaxStages, st));
}

// log2 of the elements per tile: one slot of the task's widest operand (fp32
// wire tasks have fp32 results, whose tile goes back over input 0's slot)
__device__ __forceinline__ int rt_te_lg(const DTask* tk, int slot_lg) { return slot_lg - (tk->out_f32 ? 2 : 1); }

__device__ __forceinline__ bool rt_tile(const RoundsArgs& a, const DRound& rd, int64_t t, int slot_lg,
                                        const DTask*& task, int64_t& e0, int& ne) {
  for (int ti = rd.t0; ti < rd.t1; ++ti) {
    const DTask* tk = a.tasks + ti;
    if (tk->nin > kRtMaxIn) continue;
    const int lg = rt_te_lg(tk, slot_lg);
    const int64_t n = tk->n8 * 8;
    const int64_t nt = (n + (1ll << lg) - 1) >> lg;
    if (t < nt) {
      task = tk;
      e0 = t << lg;
      ne = (int)min((int64_t)1 << lg, n - e0);
      return true;
    }
    t -= nt;
  }
  return false;
}

// One tile of an fp32-wire task (fp32 result) or a nested fold (one-shot
// topology), from the stage `base`: nblk blocks of nest inputs, each folded in
// order, then the block results, then the remaining inputs; on the task's wire
// (fp32 adds, or the bf16 hop).  bulk: the result goes back over input 0's slot
// (the fp32 result is wider than a bf16 input: every thread reads first).
__device__ __forceinline__ void rt_fold_generic(const DTask* tk, unsigned char* base, int slotb, int ne, int64_t e0,
                                                float alpha, bool bulk) {
  const bool wide = tk->out_f32 != 0;
  const int nin = tk->nin;
  const uint32_t raw = tk->rawmask, f32 = tk->f32mask;
  const int nest = tk->nest > 1 ? tk->nest : nin, nblk = tk->nest > 1 ? tk->nblk : 1;
  const int nu = ne / 8;
  for (int u0 = 0; u0 < nu; u0 += kRtThreads) {   // wide tiles: one pass (<= 256 units)
    const int u = u0 + threadIdx.x;
    const bool act = u < nu;
    float acc[8];
    if (act) {
      auto ld = [&](int i, float x[8]) {
        if ((f32 >> i) & 1u) {
          const float4* q = reinterpret_cast<const float4*>(base + i * slotb) + 2 * u;
          f4x2(q[0], q[1], x);
        } else {
          unpack8(reinterpret_cast<const uint4*>(base + i * slotb)[u], x);
          if ((raw >> i) & 1u) pre8(x, alpha, wide);
        }
      };
      int i = 0;
      for (int b = 0; b < nblk; ++b) {
        float blk[8];
        ld(i++, blk);
        for (int q = 1; q < nest; ++q) {
          float x[8];
          ld(i++, x);
          hopw8(blk, x, wide);
        }
        if (b == 0) {
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[e] = blk[e];
        } else {
          hopw8(acc, blk, wide);
        }
      }
      for (; i < nin; ++i) {
        float x[8];
        ld(i, x);
        hopw8(acc, x, wide);
      }
    }
    if (wide) {
      if (bulk) {
        __syncthreads();
        if (act) {
          float4* q = reinterpret_cast<float4*>(base) + 2 * u;
          q[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
          q[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
        }
      } else if (act) {
        float4* q = reinterpret_cast<float4*>(tk->dst) + (e0 / 8 + u) * 2;
        __stcg(q, make_float4(acc[0], acc[1], acc[2], acc[3]));
        __stcg(q + 1, make_float4(acc[4], acc[5], acc[6], acc[7]));
      }
    } else if (act) {
      if (bulk) reinterpret_cast<uint4*>(base)[u] = pack8(acc);   // same width: in place, this thread read it
      else __stcg(reinterpret_cast<uint4*>(tk->dst + e0) + u, pack8(acc));
    }
  }
}

// kBulk: the folded tile goes back into its shared-memory stage (in place over
// input 0) and leaves through one cp.async.bulk global<-shared per tile (the
// bulk-copy engine keeps the NVLink stores of the push transport in flight
// without LSU slots); the stage is refilled one tile later, after
// wait_group.read, and every bulk store has completed before the next peer
// barrier publishes the round.
// <= 64 registers (launch bounds 256 x 4): a rounds CTA (256 x 64) must fit
// beside a 512-thread Adam CTA (512 x <= 84: launch bounds (512, 1)) in the SM's 64 K
// registers, so collectives and updates co-run
// kGen: the launch has fp32-wire or nested (one-shot) tasks; their folds are
// compiled into a separate instantiation so the common bf16 path keeps every
// value in registers (<= 64, no spills).
template <bool kBulk, bool kGen>
__global__ void __launch_bounds__(kRtThreads, 4) rounds_tma_kernel(const RoundsArgs a, int max_in, int slot_lg,
                                                                   int nst) {
  const int slotb = 1 << slot_lg;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bars[kRtMaxStages];
  if (a.bar.err && *(volatile int*)a.bar.err) return;   // sticky device error: do nothing
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t stage_bytes = (size_t)max_in * slotb;
  uint32_t cnt = 0;   // tiles this CTA has consumed so far (stage = cnt % S, parity = cnt / S)
  int bidx = 0, narr = 0;
  unsigned long long mi = 0, me = 0;   // NVLink bytes of the tiles this CTA issued (thread 0)
  const uint64_t gen0 = launch_gen(a);
  trace_stamp(a, 0);
  for (int r = 0; r < a.nrounds; ++r) {
    const DRound rd = a.rounds[r];
    if (a.bar.my_flags && !launch_barrier(a, rd.peers_before, bidx, narr, gen0)) return;
    // order the peers' released (generic-proxy) writes before our async-proxy reads
    if (threadIdx.x == 0) asm volatile("fence.proxy.async;" ::: "memory");
    trace_stamp(a, 1 + 2 * r);
    int64_t total = 0;
    for (int ti = rd.t0; ti < rd.t1; ++ti) {
      const DTask* tk = a.tasks + ti;
      if (tk->nin <= kRtMaxIn) {
        const int lg = rt_te_lg(tk, slot_lg);
        total += (tk->n8 * 8 + (1ll << lg) - 1) >> lg;
      }
    }
    const int64_t mine = (total > blockIdx.x) ? (total - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const uint64_t t_round = globaltimer();
    double inter_sent = 0.0;   // bytes of inter-group tiles this CTA has issued in this round
    auto issue = [&](int64_t k) {
      const DTask* tk;
      int64_t e0;
      int ne;
      rt_tile(a, rd, blockIdx.x + k * gridDim.x, slot_lg, tk, e0, ne);
      if (tk->inter && a.inter_bytes_per_ns > 0.0) {   // token bucket: emulated slow inter link
        inter_sent += (double)ne * (tk->out_f32 ? 4.0 : 2.0) * (double)tk->inter;
        while (inter_sent > (double)(globaltimer() - t_round) * a.inter_bytes_per_ns) __nanosleep(256);
      }
      count_moved(tk, ne, mi, me);
      const uint32_t slot = (cnt + (uint32_t)k) % nst;
      unsigned char* base = smem + slot * stage_bytes;
      uint32_t tx = 0;
      for (int i = 0; i < tk->nin; ++i) tx += (uint32_t)ne * (((tk->f32mask >> i) & 1u) ? 4 : 2);
      mbar_expect_tx(&bars[slot], tx);
      for (int i = 0; i < tk->nin; ++i) {
        const int es = ((tk->f32mask >> i) & 1u) ? 4 : 2;
        bulk_g2s(base + i * slotb, reinterpret_cast<const unsigned char*>(tk->in[i]) + (size_t)e0 * es,
                 (uint32_t)ne * es, &bars[slot]);
      }
    };
    if (threadIdx.x == 0)
      for (int64_t k = 0; k < min((int64_t)nst, mine); ++k) issue(k);
    for (int64_t k = 0; k < mine; ++k) {
      const uint32_t c = cnt + (uint32_t)k;
      const uint32_t slot = c % nst;
      mbar_wait(&bars[slot], (c / nst) & 1u);
      const DTask* tk;
      int64_t e0;
      int ne;
      rt_tile(a, rd, blockIdx.x + k * gridDim.x, slot_lg, tk, e0, ne);
      unsigned char* base = smem + slot * stage_bytes;
      const int nin = tk->nin;
      const uint32_t raw = tk->rawmask;
      const int osz = tk->out_f32 ? 4 : 2;
      if (kGen && (tk->out_f32 || tk->nest > 1)) {
        rt_fold_generic(tk, base, slotb, ne, e0, a.alpha, kBulk);   // fp32-wire or nested tile
      } else {
        uint4* dst = reinterpret_cast<uint4*>(tk->dst + e0);
        for (int u = threadIdx.x; u < ne / 8; u += kRtThreads) {
          const uint4 v0 = reinterpret_cast<const uint4*>(base)[u];
          if (nin == 1 && !(raw & 1u)) {   // plain copy: the stage already holds the result
            if (!kBulk) __stcg(dst + u, v0);
            continue;
          }
          float acc[8];
          unpack8(v0, acc);
          if (raw & 1u) scale_round8(acc, a.alpha);
          for (int i = 1; i < nin; ++i) {
            float x[8];
            unpack8(reinterpret_cast<const uint4*>(base + i * slotb)[u], x);
            if ((raw >> i) & 1u) scale_round8(x, a.alpha);
            hop8(acc, x);
          }
          if (kBulk) reinterpret_cast<uint4*>(base)[u] = pack8(acc);   // in place: this thread read it
          else __stcg(dst + u, pack8(acc));
        }
      }
      if (kBulk) {
        fence_proxy_async_smem();   // this thread's smem writes -> visible to the bulk-copy engine
        __syncthreads();
        if (threadIdx.x == 0) {
          bulk_s2g(reinterpret_cast<unsigned char*>(tk->dst) + (size_t)e0 * osz, base, (uint32_t)ne * osz);
          bulk_commit();
          bulk_wait_read<1>();      // the previous tile's store has read its stage: refill it
          if (k >= 1 && k - 1 + nst < mine) issue(k - 1 + nst);
        }
      } else {
        __syncthreads();   // stage consumed by every thread: refill it
        if (threadIdx.x == 0 && k + nst < mine) issue(k + nst);
      }
    }
    cnt += (uint32_t)mine;
    if (kBulk && threadIdx.x == 0) {   // the round's stores are complete (and the stages free)
      bulk_wait_all();                 // before anyone reads them or the next round reuses
      asm volatile("fence.proxy.async.global;" ::: "memory");   // the stages
    }
    __syncthreads();
    trace_stamp(a, 2 + 2 * r);
  }
  if (a.bar.my_flags && a.final_barrier && !launch_barrier(a, a.final_peers, bidx, narr, gen0)) return;
  if (threadIdx.x == 0) flush_moved(a.moved, mi, me);
  launch_exit(a, gen0);
  trace_stamp(a, kTraceSlots - 1);
}

// ------------------------------------------------------------- two-phase step (R28)
// Phase 1: sum (fold(gin) * s_g)^2 and the non-finite flag over the segments,
// same partition and block reduction as adam_kernel (2 B read per element).
__global__ void __launch_bounds__(kAdamBlock) grad_norm_kernel(const AdamArgs a) {
  int64_t U = 0;
  for (int i = 0; i < a.nseg; ++i) U += a.seg[i].n8;
  const int64_t per = (U + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = min(U, (int64_t)blockIdx.x * per);
  const int64_t b1 = min(U, b0 + per);
  double nsq = 0.0;
  int bad = 0;
  int64_t base = 0;
  for (int i = 0; i < a.nseg && base < b1; ++i) {
    const AdamSeg& sg = a.seg[i];
    const int64_t n8 = sg.n8;
    const int64_t s = max(b0, base) - base, e = min(b1, base + n8) - base;
    if (sg.in_norm) {
      for (int64_t u = s + threadIdx.x; u < e; u += blockDim.x) {
        float g[8];
        ld_gin8(sg, 0, u, a.alpha, g);
        for (int k = 1; k < sg.gnin; ++k) {
          float x[8];
          ld_gin8(sg, k, u, a.alpha, x);
          hopw8(g, x, sg.gwide != 0);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (!isfinite(g[q])) bad = 1;
          const float gr = __fmul_rn(g[q], a.s_g);
          nsq += (double)gr * (double)gr;
        }
      }
    }
    base += n8;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nsq += __shfl_xor_sync(0xffffffffu, nsq, o);
  __shared__ double s_part[kAdamBlock / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) s_part[wid] = nsq;
  const int any_bad = __syncthreads_or(bad);
  if (wid == 0) {
    double x = (lane < (int)(blockDim.x / 32)) ? s_part[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) {
      a.partials[blockIdx.x] = x;
      if (any_bad) atomicOr(a.nonfinite, 1);
    }
  }
}

__global__ void clip_scale_kernel(const double* norm_sq, const int* nonfinite, double clip, double base,
                                  int skip_nonfinite, float* s_g_out, int* skip_out) {
  const double n = sqrt(*norm_sq);
  double coef = 1.0;
  if (clip > 0.0 && isfinite(n)) coef = fmin(1.0, clip / (n + 1e-6));
  *s_g_out = (float)(base * coef);
  *skip_out = (skip_nonfinite && *nonfinite) ? 1 : 0;
}

// ------------------------------------------------------------- norm finalize
__global__ void __launch_bounds__(1024) norm_finalize_kernel(const double* p, int n, double* out) {
  __shared__ double sh[1024];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += p[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = sh[0];
}

// ------------------------------------------------------------- pack / copy
__global__ void __launch_bounds__(256) pack_kernel(const PackEntry* table) {
  const PackEntry e = table[blockIdx.y];
  const bool vec = (((uintptr_t)e.src | (uintptr_t)e.dst) & 15) == 0;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (vec) {
    const int64_t n8 = e.n / 8;
    const uint4* s = reinterpret_cast<const uint4*>(e.src);
    uint4* d = reinterpret_cast<uint4*>(e.dst);
    for (int64_t i = tid; i < n8; i += nth) d[i] = __ldcs(s + i);
    done = n8 * 8;
  }
  for (int64_t i = done + tid; i < e.n; i += nth) e.dst[i] = e.src[i];
}

// ------------------------------------------------------------- synthetic inputs
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint16_t synth_grad_bits(uint64_t key, uint64_t i) {
  const uint64_t h = splitmix64(key ^ i);
  const uint32_t sign = (uint32_t)(h >> 63);
  const uint32_t expo = 114u + (uint32_t)((h >> 8) % 5ull);
  const uint32_t mant = (uint32_t)((h >> 16) & 0x7Full);
  return (uint16_t)((sign << 15) | (expo << 7) | mant);
}

__device__ __forceinline__ float synth_master(uint64_t key, uint64_t i) {
  const uint64_t h = splitmix64(key ^ i);
  const uint32_t sign = (uint32_t)(h >> 63);
  const uint32_t expo = 119u + (uint32_t)((h >> 8) % 5ull);
  const uint32_t mant = (uint32_t)(h & 0x7FFFFFull);
  return __uint_as_float((sign << 31) | (expo << 23) | mant);
}

// dst[k] = gradient of flat element begin + k, k < n (n, begin multiples of 8)
__global__ void synth_grad_kernel(uint16_t* dst, int64_t begin, int64_t n, int64_t psi, uint64_t key) {
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n / 8; u += nth) {
    uint16_t b[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int64_t i = begin + u * 8 + e;
      b[e] = (i < psi) ? synth_grad_bits(key, (uint64_t)i) : (uint16_t)0;
    }
    uint4 v;
    v.x = b[0] | ((uint32_t)b[1] << 16); v.y = b[2] | ((uint32_t)b[3] << 16);
    v.z = b[4] | ((uint32_t)b[5] << 16); v.w = b[6] | ((uint32_t)b[7] << 16);
    reinterpret_cast<uint4*>(dst)[u] = v;
  }
}

__global__ void init_range_kernel(const float* src, uint64_t key, int64_t begin, int64_t n, int64_t psi,
                                  float* master, float* m, float* v, uint16_t* pdst) {
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += nth) {
    const int64_t f = begin + i;
    float val = 0.f;
    if (f < psi) val = src ? src[f] : synth_master(key, (uint64_t)f);
    if (master) {
      master[i] = val;
      m[i] = 0.f;
      v[i] = 0.f;
    }
    if (pdst) {
      __nv_bfloat16 b = __float2bfloat16_rn(val);
      pdst[i] = *reinterpret_cast<uint16_t*>(&b);
    }
  }
}

}  // namespace

// ------------------------------------------------------------- launchers
int adam_grid() { return 148 * 8; }
int adam_block() { return kAdamBlock; }

// All kernels that may share an SM prefer the maximum shared-memory carveout,
// so the SM never has to drain to re-split L1/shared between a collective CTA
// and an Adam CTA.
static cudaError_t set_carveouts() {
  static bool done = false;
  if (done) return cudaSuccess;
  const void* fns[] = {(const void*)rounds_kernel, (const void*)rounds_tma_kernel<false, false>,
                       (const void*)rounds_tma_kernel<true, false>, (const void*)rounds_tma_kernel<false, true>,
                       (const void*)rounds_tma_kernel<true, true>, (const void*)adam_kernel,
                       (const void*)adam_tma_kernel<false, 512, false>, (const void*)adam_tma_kernel<true, 512, false>,
                       (const void*)adam_tma_kernel<true, 256, false>, (const void*)adam_tma_kernel<false, 256, false>,
                       (const void*)adam_tma_kernel<false, 512, true>, (const void*)adam_tma_kernel<true, 512, true>,
                       (const void*)adam_tma_kernel<true, 256, true>, (const void*)adam_tma_kernel<false, 256, true>,
                       (const void*)adam_tma_ws_kernel<512, false>, (const void*)adam_tma_ws_kernel<256, false>,
                       (const void*)adam_tma_ws_kernel<512, true>, (const void*)adam_tma_ws_kernel<256, true>};
  for (const void* f : fns) {
    cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout,
                                         (int)cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
  }
  done = true;
  return cudaSuccess;
}

cudaError_t launch_rounds(const RoundsArgs& a, int grid, int block, cudaStream_t s) {
  cudaError_t e = set_carveouts();
  if (e != cudaSuccess) return e;
  rounds_kernel<<<grid, block > 0 ? block : kRoundsBlock, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_rounds_tma(const RoundsArgs& a, int grid, int max_in, cudaStream_t s, int bulk_store,
                              int generic) {
  cudaError_t ec = set_carveouts();
  if (ec != cudaSuccess) return ec;
  static bool attr_set = false;
  if (!attr_set) {
    for (const void* f : {(const void*)rounds_tma_kernel<false, false>, (const void*)rounds_tma_kernel<true, false>,
                          (const void*)rounds_tma_kernel<false, true>, (const void*)rounds_tma_kernel<true, true>}) {
      cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, kRtSmem);
      if (e != cudaSuccess) return e;
    }
    attr_set = true;
  }
  if (max_in < 1) max_in = 1;
  if (max_in > kRtMaxIn) max_in = kRtMaxIn;
  const int lg = rt_slot_lg(max_in);
  const int nst = rt_stages(max_in);
  const size_t sm = (size_t)nst * max_in << lg;
  if (generic) {
    if (bulk_store) rounds_tma_kernel<true, true><<<grid, kRtThreads, sm, s>>>(a, max_in, lg, nst);
    else rounds_tma_kernel<false, true><<<grid, kRtThreads, sm, s>>>(a, max_in, lg, nst);
  } else {
    if (bulk_store) rounds_tma_kernel<true, false><<<grid, kRtThreads, sm, s>>>(a, max_in, lg, nst);
    else rounds_tma_kernel<false, false><<<grid, kRtThreads, sm, s>>>(a, max_in, lg, nst);
  }
  return cudaGetLastError();
}

int rounds_tma_smem_kb(int max_in) {
  if (max_in < 1) max_in = 1;
  if (max_in > kRtMaxIn) max_in = kRtMaxIn;
  return (rt_stages(max_in) * max_in * rt_slot_bytes(max_in) + 1023) / 1024;
}

cudaError_t launch_adam(const AdamArgs& a, int grid, cudaStream_t s, int cap_two_per_sm) {
  cudaError_t ec = set_carveouts();
  if (ec != cudaSuccess) return ec;
  // With collectives running concurrently, Adam is capped at two CTAs per SM
  // (an 80 KB shared-memory reservation) so a 512-thread collective CTA always
  // fits beside it (registers: 2 x 256 x 80 + 512 x 48 = 64K).
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(adam_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  adam_kernel<<<grid, kAdamBlock, cap_two_per_sm ? 80 * 1024 : 0, s>>>(a);
  return cudaGetLastError();
}

// warp-specialized TMA-store Adam (adam_tma_ws_kernel); PARO_ADAM_WS=0/1 for A/B
bool adam_ws_on() {
  static const int env = std::getenv("PARO_ADAM_WS") ? std::atoi(std::getenv("PARO_ADAM_WS")) : -1;
  return env == 1;
}

// TMA pipeline: persistent grid (one CTA per SM), stages sized to the budget.
// smem_budget_kb sets the stage count (2-4); hard_kb is what the SM can give
// Adam beside the co-running collective CTA (its stages are the rest of the
// 228 KB).  Thread stores (kStore = false) keep >= 2 stages of 4096-element
// tiles (512 threads) when they fit hard_kb, else 2048-element tiles (256
// threads).  The TMA-store variant refills a stage one iteration late (after
// its stores have read it), so it keeps >= 3 stages: with a small budget it
// switches to 2048-element tiles.  Returns the variant (AdamVariant) and stage
// count through *variant / *stages.
cudaError_t launch_adam_tma(const AdamArgs& a, int sms, cudaStream_t s, int smem_budget_kb, int tma_store,
                            int hard_kb, int* variant, int* stages, int ws) {
  cudaError_t ec = set_carveouts();
  if (ec != cudaSuccess) return ec;
  int gmax = 1, gsz = 2;
  for (int i = 0; i < a.nseg; ++i) {
    gmax = a.seg[i].gnin > gmax ? a.seg[i].gnin : gmax;
    // fp32 wire: fp32 arithmetic even when every input is a raw bf16 gradient
    // (a fused one-shot hop or the fused all-reduce at M = 1), 4-byte slots
    if (a.seg[i].gf32 || a.seg[i].gwide) gsz = 4;
  }
  static bool attr_set = false;
  if (!attr_set) {
    for (const void* f : {(const void*)adam_tma_kernel<false, 512, false>, (const void*)adam_tma_kernel<true, 512, false>,
                          (const void*)adam_tma_kernel<true, 256, false>, (const void*)adam_tma_kernel<false, 256, false>,
                          (const void*)adam_tma_kernel<false, 512, true>, (const void*)adam_tma_kernel<true, 512, true>,
                          (const void*)adam_tma_kernel<true, 256, true>, (const void*)adam_tma_kernel<false, 256, true>,
                          (const void*)adam_tma_ws_kernel<512, false>, (const void*)adam_tma_ws_kernel<256, false>,
                          (const void*)adam_tma_ws_kernel<512, true>, (const void*)adam_tma_ws_kernel<256, true>}) {
      cudaError_t e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
      if (e != cudaSuccess) return e;
    }
    attr_set = true;
  }
  if (hard_kb <= 0 || hard_kb > 220) hard_kb = 220;
  auto stage_bytes = [&](int tile) { return (size_t)tile * (gsz * gmax + 12); };
  auto raw = [&](int tile, int kb) { return (int)(((size_t)kb * 1024) / stage_bytes(tile)); };
  auto clampst = [](int st, int lo) { return st > 4 ? 4 : (st < lo ? lo : st); };
  const bool wide = gsz == 4;
#define PARO_ADAM_WS_LAUNCH(KT)                                                                          \
  do {                                                                                                   \
    if (wide) adam_tma_ws_kernel<KT, true><<<sms, KT + 32, stage_bytes(KT * 8) * st, s>>>(a, gmax, st);  \
    else adam_tma_ws_kernel<KT, false><<<sms, KT + 32, stage_bytes(KT * 8) * st, s>>>(a, gmax, st);      \
  } while (0)
#define PARO_ADAM_LAUNCH(KS, KT)                                                                    \
  do {                                                                                              \
    if (wide) adam_tma_kernel<KS, KT, true><<<sms, KT, stage_bytes(KT * 8) * st, s>>>(a, gmax, st); \
    else adam_tma_kernel<KS, KT, false><<<sms, KT, stage_bytes(KT * 8) * st, s>>>(a, gmax, st);     \
  } while (0)
  int v = 0, st = 0;
  if (!tma_store) {
    st = clampst(raw(4096, smem_budget_kb), 2);
    if ((size_t)st * stage_bytes(4096) <= (size_t)hard_kb * 1024) {
      v = ADAM_TMA_LD_512;
      PARO_ADAM_LAUNCH(false, 512);
    } else {
      st = clampst(std::min(raw(2048, smem_budget_kb), raw(2048, hard_kb)), 2);
      v = ADAM_TMA_LD_256;
      PARO_ADAM_LAUNCH(false, 256);
    }
  } else if (raw(4096, smem_budget_kb) >= 3) {
    st = clampst(raw(4096, smem_budget_kb), 3);
    if (ws == 1 || (ws < 0 && adam_ws_on())) {
      v = ADAM_TMA_WS_512;
      PARO_ADAM_WS_LAUNCH(512);
    } else {
      v = ADAM_TMA_ST_512;
      PARO_ADAM_LAUNCH(true, 512);
    }
  } else {
    st = clampst(raw(2048, smem_budget_kb), 3);
    if (ws == 1 || (ws < 0 && adam_ws_on())) {
      v = ADAM_TMA_WS_256;
      PARO_ADAM_WS_LAUNCH(256);
    } else {
      v = ADAM_TMA_ST_256;
      PARO_ADAM_LAUNCH(true, 256);
    }
  }
#undef PARO_ADAM_LAUNCH
#undef PARO_ADAM_WS_LAUNCH
  if (variant) *variant = v;
  if (stages) *stages = st;
  return cudaGetLastError();
}

cudaError_t launch_norm_finalize(const double* partials, int n, double* out, cudaStream_t s) {
  norm_finalize_kernel<<<1, 1024, 0, s>>>(partials, n, out);
  return cudaGetLastError();
}

cudaError_t launch_grad_norm(const AdamArgs& a, int grid, cudaStream_t s) {
  grad_norm_kernel<<<grid, kAdamBlock, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_clip_scale(const double* norm_sq, const int* nonfinite, double clip, double base,
                              int skip_nonfinite, float* s_g_out, int* skip_out, cudaStream_t s) {
  clip_scale_kernel<<<1, 1, 0, s>>>(norm_sq, nonfinite, clip, base, skip_nonfinite, s_g_out, skip_out);
  return cudaGetLastError();
}

cudaError_t launch_pack(const PackEntry* table, int n_entries, int64_t max_n, cudaStream_t s) {
  if (n_entries <= 0) return cudaSuccess;
  int64_t bx = (max_n / 8 + 255) / 256;
  if (bx < 1) bx = 1;
  if (bx > 512) bx = 512;
  dim3 grid((unsigned)bx, (unsigned)n_entries);
  pack_kernel<<<grid, 256, 0, s>>>(table);
  return cudaGetLastError();
}

cudaError_t launch_synth_grad(uint16_t* dst, int64_t psi, int64_t psi_pad, uint64_t key, cudaStream_t s) {
  synth_grad_kernel<<<148 * 16, 256, 0, s>>>(dst, 0, psi_pad, psi, key);
  return cudaGetLastError();
}

cudaError_t launch_synth_grad_range(uint16_t* dst, int64_t begin, int64_t n, int64_t psi, uint64_t key,
                                    cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  synth_grad_kernel<<<148 * 16, 256, 0, s>>>(dst, begin, n, psi, key);
  return cudaGetLastError();
}

cudaError_t launch_init_range(const float* src, uint64_t key, int64_t begin, int64_t n, int64_t psi,
                              float* master, float* m, float* v, uint16_t* pdst, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  init_range_kernel<<<(unsigned)blocks, 256, 0, s>>>(src, key, begin, n, psi, master, m, v, pdst);
  return cudaGetLastError();
}

uint64_t splitmix64_host(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t synth_key(uint64_t seed, uint64_t tag, uint64_t rank, uint64_t step) {
  return splitmix64_host(splitmix64_host(seed ^ tag) ^ ((rank << 32) | step));
}

}  // namespace paro
