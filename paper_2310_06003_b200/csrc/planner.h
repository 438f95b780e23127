// planner.h — host-only PaRO planner: strategy validation, flat layout,
// buckets, position-major shard map, per-bucket collective schedule (as
// symbolic pull-model transfer lists for every rank), and byte/memory
// accounting.  No CUDA here: the planning-only context uses it on a CPU box.
//
// Paper: P = PAPER.md line.  Strategy codes and Principle 1: P:240-243,
// Table 1 P:266-298.  Shard levels N/I/G: P:185-188.  Schedules: P:333-363.
// HO-Ring: P:385-410.  Memory: Table 2 P:416-439.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace paro {

enum Level : int { LV_N = 0, LV_I = 1, LV_G = 2 };

// Buffers of one rank, all bf16, carved from one symmetric allocation so a
// (rank, kind, offset) triple names the same bytes on every rank.
enum BufKind : int {
  BUF_GRAD = 0,    // flat gradients, psi_pad (raw: scaled by 1/N when read)
  BUF_PARAM,       // parameter residency, p_numel
  BUF_GSHARD,      // gradient residency (G = I or G), g_numel
  BUF_GHAT,        // reduced-gradient slots when G != OS
  BUF_STAGE_I,     // intra-ring partials: 2 parities x 2 slots
  BUF_STAGE_E,     // inter-ring partials: 2 parities x 2 slots
  BUF_P1,          // HO phase-1 / direct phase-1 output: 2 parities
  BUF_SOWN,        // own-group partial (HO phase 2): 2 parities
  BUF_LAND,        // direct push landing slots: 2 parities x ((M-1) chunks + (g-1) segments)
  BUF_GACC,        // G = N gradient accumulator (psi_pad; only for grad_accum plans)
  BUF_WIN,         // forward/backward parameter gather windows: n_windows x B (P = I or G)
  BUF_XW,          // NCCL comparator on the fp32 wire: the bucket's pre-scaled fp32 gradients (B)
  BUF_NKINDS
};

constexpr int kMaxIn = 16;     // max inputs of one fold task
constexpr int kStageSets = 3;  // rotation of per-bucket staging sets (reuse distance)
constexpr int kMaxAdamIn = 4;  // max fold inputs of the fused final hop in Adam
constexpr int kMaxPush = 8;    // max peers one fused-gather Adam store goes to

struct Ref {
  int32_t rank = -1;
  int32_t kind = -1;
  int64_t off = 0;           // element offset inside the buffer kind
  bool raw = false;          // holds raw gradient bits (copied): scaled 1/N when read
  bool is_raw() const { return raw || kind == BUF_GRAD; }
};

// dst = (((in0 (+) in1) (+) in2) ...), (+) = RNE_bf16(fp32 + fp32); inputs
// that reference BUF_GRAD are first scaled: RNE_bf16(fp32(g) * alpha).
// nin == 1 is a copy (or a pack when the input is raw).
struct Task {
  int64_t n = 0;             // elements (multiple of 8)
  int32_t nin = 0;
  Ref in[kMaxIn];
  Ref dst;
  // nested fold (one-shot topology): the first nest * nblk inputs are nblk
  // blocks of nest; each block is folded in order, then the block results in
  // order, then any further inputs: ((b_0 (+) b_1) ...) with b_k = fold(block k)
  int32_t nest = 0, nblk = 0;
};

// One collective launch = rounds; round r holds, for every rank, its tasks.
struct Launch {
  std::vector<std::vector<std::vector<Task>>> rounds;  // [round][rank][task]
  bool final_barrier = false;   // barrier with the peers touched in the last round
  std::vector<uint64_t> final_extra;  // per rank: extra final-barrier peers (fused Adam reads)
  std::vector<uint64_t> first_extra;  // per rank: extra round-0 barrier peers (their fused Adam
                                      // read the slot this launch overwrites)
  int n_ranks = 0;
  void add(int round, int rank, const Task& t);
  bool empty() const { return rounds.empty() && !final_barrier; }
  // other ranks whose memory `rank` reads or writes in round r
  std::vector<int> reads(int r, int rank) const;
  // symmetric barrier peer set before round r (r == rounds.size(): final)
  uint64_t barrier_peers(int r, int rank) const;
};

// NCCL comparator call (PARO_TOPO_NCCL): not bit-exact, perf only.
struct NcclCall {
  enum Kind { RS, AG, AR } kind;
  enum Comm { WORLD, INTRA, INTER } comm;
  Ref send, recv;            // for the local rank (rank field = owner)
  int64_t count;             // recv count (RS), send count (AG), count (AR)
};

struct BucketSchedule {
  Launch reduce;             // gradient reduction to the OS residency
  Launch gather;             // parameter restore to the P residency
  std::vector<std::vector<NcclCall>> nccl_reduce, nccl_gather;  // [rank][call]
  // Adam input/output per rank for this bucket
  std::vector<Ref> ghat;     // reduced gradient at the OS residency start
  // Adam's g_hat = fold(ghat_in[r]) (1 input = materialised g_hat; up to 3 when
  // the final reduction hop is fused into the Adam kernel)
  std::vector<std::vector<Ref>> ghat_in;
  std::vector<Ref> param;    // parameter-buffer position of the OS residency
  std::vector<int64_t> os_off;   // offset in the rank's opt-state arrays
  int64_t os_len = 0;
  // gradient accumulation (R27): `accum` reduces one micro-batch to
  // the G residency and writes the accumulator (the engine appends the
  // accumulator as the last fold input from the second micro-batch on);
  // `reduce_acc` finishes the reduction from the accumulator after the last one
  Launch accum, reduce_acc;
  std::vector<std::vector<Ref>> ghat_in_acc;
  // forward/backward parameter all-gather of the whole bucket into window slot
  // 0; the engine shifts BUF_WIN refs to the slot used
  Launch window;
  // fused parameter all-gather: Adam also stores its bf16 output into these
  // peers' parameter buffers (same offset: the layouts are symmetric), which
  // replaces the gather launch when the consumers are one ring's members
  std::vector<std::vector<Ref>> param_push;
  // copy-engine transport (opt.ce_reduce): raw gradient chunks of the group
  // peers copied into landing slots before `reduce` / `accum` fold them locally
  Launch reduce_pre, accum_pre;
};

struct PlanOptions {
  int64_t bucket_elems = int64_t(1) << 26;
  int topology = 0;          // PARO_TOPO_*
  int pipeline_depth = 2;
  bool push = true;          // push (remote stores) or pull (remote loads) transport
  bool fuse_final = true;    // OS = G: fold the owner's last reduction hop into Adam
  bool fuse_ar_e = true;     // OS = I, G = I, g = 2 (pull): AR_E folded into Adam (R31)
  bool accum = false;        // build the gradient-accumulation launches (s > 1)
  bool two_phase = false;    // clipping / skip: every bucket's g_hat stays resident until Adam (R28)
  int windows = 0;           // parameter-gather window slots (0: none)
  bool ce_reduce = false;    // G = I: RS_I as copy-engine copies of raw chunks + one local fold
  int grad_slots = 0;        // > 0: raw gradients live in this many bucket slots (slot b % K)
                             // filled by a producer as the step streams, not in one psi_pad buffer
  bool params_only = false;  // frozen tensors (partial / PEFT training): only
                             // the parameter residency and its forward/backward gathers
  int fuse_gather = 1;       // fold a one-ring parameter all-gather into Adam's stores:
                             // 0 never, 1 when no collective rounds co-run, 2 always
  int wire = 2;              // bytes per reduction element on the wire and in the G / g_hat /
                             // staging buffers: 2 = bf16, 4 = fp32 (reading A3)
  bool predivide = true;     // raw gradients scaled by 1/N when first read (R4); else in Adam
  std::vector<int64_t> groups;   // layer-aligned buckets: tensor indices starting a bucket
                                 // (first 0); each bucket padded at its end to N*64 (NEXT-2)
};

class Planner {
 public:
  // Throws std::invalid_argument with the user-facing message.
  Planner(int N, int M, const std::string& code, const std::vector<int64_t>& sizes,
          const PlanOptions& opt);

  int N, M, g;
  Level P, G, OS;
  std::string code;
  PlanOptions opt;
  int64_t psi = 0, psi_pad = 0, B = 0;
  bool fused_allreduce = false;   // the inter all-reduce runs inside Adam (R31)
  std::vector<std::pair<int64_t, int64_t>> buckets;   // (start, size)
  std::vector<int64_t> bucket_real_end;               // end of the real (non-padding) elements per bucket
  std::vector<int64_t> param_sizes, param_offsets;
  int64_t p_numel = 0, g_numel = 0, os_numel = 0;
  int nslots = 0;                                      // BUF_GHAT slots
  int64_t ghat_slot = 0;                               // elements per slot
  int64_t buf_len[BUF_NKINDS] = {0};                   // elements per kind
  int64_t buf_off[BUF_NKINDS] = {0};                   // BYTE offset of each kind in the region
  int esz[BUF_NKINDS] = {0};                           // bytes per element of each kind
  int64_t region_bytes = 0;                            // symmetric region (after the header)
  int64_t stage_i_len = 0, stage_e_len = 0, p1_len = 0, sown_len = 0, land_len = 0;

  std::vector<BucketSchedule> sched;
  std::vector<std::string> grad_ops, rest_ops;        // primitives (for reporting)
  std::vector<int64_t> send_intra, send_inter;        // bytes per rank per step
  std::vector<int64_t> acc_send_intra, acc_send_inter;        // per accumulated micro-batch
  std::vector<int64_t> accstep_send_intra, accstep_send_inter;  // per step after accumulation
  std::vector<int64_t> win_send_intra, win_send_inter;          // per gather of every bucket once
  std::vector<std::vector<int64_t>> win_bucket_intra, win_bucket_inter;   // [bucket][rank]: one window gather
  int acc_kind = -1;                                  // accumulator buffer (GSHARD / GACC)
  int n_rounds = 0, n_comm_launches = 0;

  static int div(Level l, int N, int M) { return l == LV_N ? 1 : (l == LV_I ? M : N); }
  int divl(Level l) const { return div(l, N, M); }
  int rank_of(int j, int p) const { return j * M + p; }
  int grp(int r) const { return r / M; }
  int pos(int r) const { return r % M; }
  int seg(int j, int p) const { return p * g + j; }

  // flat [begin, end) of `level` residency of rank r in bucket b (R1)
  void residency(Level l, int r, int64_t b, int64_t* begin, int64_t* end) const;
  int64_t mem_bytes(int state) const;   // 0 P, 1 G, 2 OS (Table 2 at psi_pad)

 private:
  void layout();
  void build_schedule();
  void count_bytes();
  void validate_refs() const;
};

Level parse_level(char c);
// Validation helpers shared by the C API (messages follow S:63).
std::string validate_strategy(const std::string& code);   // "" if OK
std::string validate_cluster(int N, int M);               // "" if OK

}  // namespace paro
