// kernels.h — device-side descriptors and launchers of the sm_100a kernels.
//
//  * rounds kernel: executes a collective's rounds of fold tasks
//      dst = (((in0 (+) in1) (+) in2) ...),  a (+) b = RNE_bf16(fp32 a + fp32 b)
//    reading peers' buffers over NVLink (real mode) with a grid + peer-flag
//    barrier between rounds; or one round per launch over all emulated ranks.
//  * adam kernel: fused unscale + fp32-master Adam + RNE bf16 cast into the
//    parameter / all-gather buffer + fp64 grad-norm partials (warp shuffles),
//    28 B of HBM traffic per element.
//  * pack / unpack, norm finalize, synthetic inputs.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace paro {

constexpr int kDevMaxIn = 16;
constexpr int kMaxAdamSegs = 16;  // emulated ranks per Adam launch
constexpr int kHeaderBytes = 4096;   // per-rank region header: flags + counters

struct DTask {
  const uint16_t* in[kDevMaxIn];   // element pointers (bf16, or fp32 where f32mask says so)
  uint16_t* dst;
  int64_t n8;        // 8-element units (16 B of bf16, 32 B of fp32)
  int32_t nin;
  uint32_t rawmask;  // bit i: input i is a raw bf16 gradient -> g * alpha (RNE_bf16 on the bf16 wire)
  int32_t inter;     // operands (inputs + dst) on another group's GPU: paced by inter_gbps
  uint32_t f32mask;  // bit i: input i holds fp32 values (fp32 wire, reading A3)
  int32_t out_f32;   // 1: fp32 wire task: fp32 arithmetic (no bf16 rounding), fp32 result
  int16_t nest, nblk;   // nested fold: nblk blocks of nest inputs, each folded, then the
                        // block results, then the remaining inputs (one-shot topology)
  uint32_t peermask;    // bit i: input i lives on another rank (pulled over NVLink)
  uint32_t intermask;   // bit i: ... on another group's rank
  int32_t dst_peer;     // result stored into another rank: 1 same group, 2 other group (push)
  int16_t mv_intra, mv_inter;   // NVLink bytes per element this task moves (pulls + push), by link class
};

struct DRound {
  int32_t t0, t1;        // task range
  int64_t units;         // sum of n8
  uint64_t peers_before; // barrier peer mask before this round (real mode)
};

// Region header layout (bytes), channel 0 (collective launches): [0, 512) uint64
// flags[64] indexed by sender; [512] arrive; [520] int32 error word; [528] go;
// [536] launch generation; [544] exit count.  Channel 2 (copy-engine barriers)
// at [1024, 1536) flags, [1536] arrive, [1544] go, [1552] generation, [1560] exit.
struct BarrierCtx {
  uint64_t* const* peer_slot;   // [N] device array: &flags_of_peer_x[me]
  uint64_t* my_flags;           // NULL => emulated mode (no barriers)
  unsigned long long* arrive;   // grid arrivals of the running launch (reset to 0 when it exits)
  unsigned long long* go;       // opened by the last-arriving CTA once the peers' flags are in
  int* err;
  unsigned long long* gen;      // launch generation of this channel: every launch reads it at start
                                // and the last CTA to exit advances it (device-resident, so
                                // launches need no host bookkeeping and can be graph-replayed)
  unsigned int* exitc;          // CTAs of the running launch that have exited
};

constexpr int kTraceSlots = 64;   // per CTA per traced launch: start, (barrier exit, work end) x rounds, end

struct RoundsArgs {
  uint64_t* trace;              // profiling: [gridDim][kTraceSlots] globaltimer stamps, or NULL
  const DRound* rounds;
  const DTask* tasks;
  int nrounds;
  int final_barrier;
  uint64_t final_peers;
  float alpha;
  double inter_bytes_per_ns;    // per-CTA pacing of inter-group tiles (0 = off)

  int sys_fence_all;            // every CTA fences at sys scope (launch stores into peer memory)
  int entry_fast;               // the launch's first barrier (no work of this launch before it) is
                                // published by CTA 0 alone, without the grid arrival
  unsigned long long* moved;    // [intra, inter] NVLink bytes this rank's CTAs pulled + pushed (or NULL)
  BarrierCtx bar;
};

constexpr int kAdamMaxIn = 4;
constexpr int kAdamMaxPush = 8;   // fused parameter all-gather: peers per store

struct AdamSeg {
  // g_hat = fold(gin[0..gnin-1]) with the hop operator: 1 input = a
  // materialised g_hat (or the raw local gradient at N = 1); 2-4 inputs =
  // the final reduction hop fused into the update (push transport, OS = G)
  const uint16_t* gin[kAdamMaxIn];
  float* master;
  float* m;
  float* v;
  uint16_t* param;
  int64_t n8;
  int32_t gnin;
  uint32_t graw;     // bit i: gin[i] is a raw gradient -> RNE_bf16(g * alpha)
  int32_t in_norm;   // elements counted in the unique-element norm
  int32_t npush;     // fused parameter all-gather: the bf16 output is also
  uint16_t* push[kAdamMaxPush];   // stored at these peer addresses (NVLink)
  uint32_t gf32;     // bit i: gin[i] holds fp32 values (fp32 wire)
  int32_t gwide;     // 1: fp32 wire: raw inputs g * alpha and hops in fp32, g_hat never rounded to bf16
  uint32_t gpeer, ginter;   // bit i: gin[i] on another rank / another group's rank (NVLink pulls)
  uint32_t pinter;          // bit i: push[i] on another group's rank (else same group)
};

struct AdamArgs {
  AdamSeg seg[kMaxAdamSegs];
  int nseg;
  float alpha;
  float b1, omb1, b2, omb2, step_size, bc2s, eps, decay, s_g;
  int has_wd;
  double* partials;  // [gridDim.x] block partial sums of (g * s_g)^2
  int* nonfinite;
  // two-phase step (clipping / non-finite skip, R28): when set, the unscale
  // factor is read from the device (computed from the global norm) and the
  // update is skipped entirely while *skip != 0
  const float* s_g_dev;
  const int* skip;
  unsigned long long* moved;   // [intra, inter] NVLink bytes pulled (fused hop) + pushed (fused gather), or NULL
};

struct PackEntry {     // one tensor slice: src/dst element pointers + count
  const uint16_t* src;
  uint16_t* dst;
  int64_t n;
};

// launchers (return cudaGetLastError())
cudaError_t launch_rounds(const RoundsArgs& a, int grid, int block, cudaStream_t s);
cudaError_t launch_adam(const AdamArgs& a, int grid, cudaStream_t s, int cap_two_per_sm);
// Adam kernel variants (reported by paro_profile_stop)
enum AdamVariant : int {
  ADAM_LSU = 0,          // adam_kernel (ld/st.global)
  ADAM_TMA_LD_512 = 1,   // adam_tma_kernel<false, 512>: bulk-copy loads, thread stores, 4096-elem tiles
  ADAM_TMA_ST_512 = 2,   // adam_tma_kernel<true, 512>: bulk-copy loads and stores
  ADAM_TMA_ST_256 = 3,   // adam_tma_kernel<true, 256>: same, 2048-elem tiles (small budget)
  ADAM_TMA_LD_256 = 4,   // adam_tma_kernel<false, 256>: thread stores, 2048-elem tiles
  ADAM_TMA_WS_512 = 5,   // adam_tma_ws_kernel<512>: bulk loads + stores, dedicated producer warp
  ADAM_TMA_WS_256 = 6    // adam_tma_ws_kernel<256>
};
// ws: 1 the warp-specialized TMA-store kernel, 0 the single-role one, -1 automatic
cudaError_t launch_adam_tma(const AdamArgs& a, int sms, cudaStream_t s, int smem_budget_kb, int tma_store,
                            int hard_kb, int* variant, int* stages, int ws);
// generic: the launch has fp32-wire (out_f32) or nested (one-shot) tasks
cudaError_t launch_rounds_tma(const RoundsArgs& a, int grid, int max_in, cudaStream_t s, int bulk_store,
                              int generic);
int rounds_tma_smem_kb(int max_in);   // dynamic shared memory of a TMA rounds CTA
cudaError_t launch_norm_finalize(const double* partials, int n, double* out, cudaStream_t s);
// phase 1 of the two-phase step: block partials of sum (fold(gin) * s_g)^2 and
// the non-finite flag, 2 bytes read per element, no update
cudaError_t launch_grad_norm(const AdamArgs& a, int grid, cudaStream_t s);
// between the phases: s_g_out = fp32(base * coef), coef = min(1, clip / (sqrt(norm_sq) + 1e-6))
// (1 if clip <= 0 or the norm is not finite); skip_out = skip_nonfinite && *nonfinite
cudaError_t launch_clip_scale(const double* norm_sq, const int* nonfinite, double clip, double base,
                              int skip_nonfinite, float* s_g_out, int* skip_out, cudaStream_t s);
cudaError_t launch_pack(const PackEntry* table, int n_entries, int64_t max_n, cudaStream_t s);
cudaError_t launch_synth_grad(uint16_t* dst, int64_t psi, int64_t psi_pad, uint64_t key, cudaStream_t s);
// gradients of flat elements [begin, begin + n) into dst (zero past psi)
cudaError_t launch_synth_grad_range(uint16_t* dst, int64_t begin, int64_t n, int64_t psi, uint64_t key,
                                    cudaStream_t s);
// init master/m/v over flat range [begin, begin+n) into os arrays at os_ptrs and
// params (bf16) at pdst (may be null); src == null => synthetic master from key
cudaError_t launch_init_range(const float* src, uint64_t key, int64_t begin, int64_t n, int64_t psi,
                              float* master, float* m, float* v, uint16_t* pdst, cudaStream_t s);
int adam_grid();
int adam_block();

// splitmix64 counter hash (paro_synth) — host copy for key derivation
uint64_t splitmix64_host(uint64_t x);
uint64_t synth_key(uint64_t seed, uint64_t tag, uint64_t rank, uint64_t step);
constexpr uint64_t kTagGrad = 0x4752414400000000ull;
constexpr uint64_t kTagMaster = 0x4D41535400000000ull;

}  // namespace paro
