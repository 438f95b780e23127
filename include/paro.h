/*
 * paro.h — C ABI of the B200-native PaRO sync + update step (libparo.so).
 *
 * PaRO (arXiv 2310.06003): N GPUs are split into g = N/M groups of M
 * (§3.1).  Each model state — parameters P, gradients G,
 * optimizer state OS — is left unsharded (N), sharded inside a group (I) or
 * sharded over all GPUs (G) (§3.1.1).  The 14 codes allowed by
 * Principle 1 (Table 1) are accepted.  One paro_step is the
 * s = 1 mini-batch update of mixed-precision Adam: reduce the bf16
 * gradients to the optimizer-state shard (intra-group reduce-scatter, inter-group
 * reduce-scatter / all-reduce, or the HO-Ring reduce-scatter, P:343, P:353-355,
 * P:385-410), run fused unscale + fp32-master Adam on the owned shard, cast to
 * bf16 into the all-gather buffer and all-gather the parameters back to their
 * residency.
 *
 * Conventions for every call
 *  - Sizes are int64_t element counts.  bf16 values are 2-byte words.
 *  - Return value is a paro_status_t.  On failure paro_last_error() returns a
 *    thread-local message valid until the next call on the same thread.
 *  - CUDA / NCCL / device-timeout failures are sticky on the context: every
 *    later call on it returns the same status until paro_finalize.
 *  - Device pointers are CUDA global-memory pointers on the context's device.
 *  - Calls on one context or plan are not thread-safe.
 *
 * Numerics (readings R2, R4-R7): gradients are pre-scaled by 1/N
 * when first read (x = RNE_bf16(g * 1/N)); every reduction hop is
 * RNE_bf16(fp32(a) + fp32(b)) in the canonical ring order; Adam is the
 * AdamW form in fp32 with IEEE-rounded operations and no FMA; the result is
 * bit-identical to unsharded data parallel for every strategy and for the
 * hierarchical topologies (HO-Ring, two-step, direct) at fixed (N, M, bucket).
 */
#ifndef PARO_H_
#define PARO_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PARO_OK = 0,
  PARO_ERR_INVALID = 1,  /* bad argument, strategy or cluster shape          */
  PARO_ERR_OOM = 2,      /* device or host allocation failed                  */
  PARO_ERR_CUDA = 3,     /* CUDA runtime error (sticky)                       */
  PARO_ERR_NCCL = 4,     /* NCCL error (sticky)                               */
  PARO_ERR_STATE = 5,    /* call not valid in this context mode / state       */
  PARO_ERR_TIMEOUT = 6   /* a device-side cross-GPU wait timed out (sticky)   */
} paro_status_t;

typedef struct paro_ctx* paro_ctx_t;
typedef struct paro_plan* paro_plan_t;

/* Opaque NCCL unique id (ncclUniqueId is 128 bytes). */
typedef struct { char bytes[128]; } paro_uid_t;

/* Caller-allocated optimizer state of one rank: three fp32 device arrays of
 * paro_plan_info_t.os_numel elements each, laid out bucket-major over the
 * rank's OS residency (DESIGN.md §4 "HBM layout").  K = 12 bytes per element
 * (Table 2). */
typedef struct { float* master; float* m; float* v; } paro_opt_state_t;

/* Topologies of the world-reaching gradient reduce-scatter / parameter
 * all-gather (used when G in {N, G}; G = I always runs RS_I then the inter op). */
enum {
  PARO_TOPO_HO_RING = 0,   /* HO-Ring: intra and inter rings overlap  */
  PARO_TOPO_TWO_STEP = 1,  /* intra ring then inter ring   */
  PARO_TOPO_FLAT_RING = 2, /* one ring over all N ranks; different bits  */
  PARO_TOPO_DIRECT = 3,    /* NVSwitch one-shot hierarchical: same bits as 0 / 1 */
  PARO_TOPO_NCCL = 4,      /* NCCL collectives on split comms: perf comparator,
                              NOT bit-exact (NCCL's reduction order)              */
  PARO_TOPO_H_RING = 5,    /* H-Ring all-gather with one leader per group (P:146-147,
                              P:401-402); its reduce-scatter runs two-step        */
  PARO_TOPO_ONESHOT = 6    /* NVSwitch one-shot, pull only: every collective is ONE
                              round (each rank reads what it needs from every peer
                              at once; RS folds in the owner's canonical nested
                              order, so same bits as 0 / 1 / 3; NNN's all-reduce
                              folds the whole bucket on every rank).  Fewest
                              barriers (small messages); more inter bytes than the
                              rings (RS / AG: (N-M)C inter per rank and bucket,
                              AR: (N-1)B).  n_gpus <= 15.                          */
};

typedef struct {
  int64_t bucket_elems;  /* default 1<<26; rounded down to a multiple of N*64     */
  int topology;          /* PARO_TOPO_*, default PARO_TOPO_HO_RING                 */
  float beta1, beta2;    /* 0.9, 0.95 (R5)                                         */
  float eps;             /* 1e-8                                                   */
  float weight_decay;    /* 0.0 (AdamW form, R5)                                   */
  float loss_scale;      /* 1.0; gradients are unscaled by 1/loss_scale in Adam    */
  int comm_ctas;         /* CTAs of the collective kernels; 0 (default): one per SM */
  int pipeline_depth;    /* buckets in flight between reduce and gather (def. 2)  */
  int pull_transport;    /* 1 (default): ranks LOAD their ring predecessor's data   *
                          * over NVLink (pull); 0: ranks STORE into their          *
                          * successor's buffers (push).  Same bits either way.     */
  int adam_impl;         /* 0 (default): TMA bulk-copy pipeline (cp.async.bulk +    *
                          * mbarrier stages; also pulls NVLink-peer operands); the *
                          * results leave through bulk copies too when N = 1 (or   *
                          * emulated, or the inter all-reduce is folded into Adam *
                          * with no collective rounds beside it and no peer       *
                          * stores: the 2 x 1 OS != G codes), through thread       *
                          * stores otherwise;                                      *
                          * 1: the LSU (ld.global) kernel; 2: TMA both ways always; *
                          * 3: TMA loads + thread stores always (the variant real  *
                          * N > 1 steps use beside collectives); 4: TMA both ways  *
                          * with a dedicated producer warp (warp-specialized).     *
                          * Same bits.                                             */
  int comm_impl;         /* 2 (default): collective rounds move operands with TMA  *
                          * bulk copies into shared memory and the folded tile     *
                          * leaves through a bulk copy too (measured 1-10 % faster *
                          * in the full step at 2x1 / 2x2, profiles/r01/           *
                          * sweep_comm_store_*.jsonl); 0: TMA loads, thread        *
                          * stores; 1: LSU kernel.  Same bits.  Other values:      *
                          * PARO_ERR_INVALID.                                      */
  float inter_gbps;      /* > 0: emulate a slow inter-group link — each rank's     *
                          * inter-group transfers are paced to this many GB/s (TMA *
                          * rounds kernel; the final hop is then not fused into    *
                          * Adam).  0 (default): no pacing.  One NVSwitch box has  *
                          * no real intra/inter gap.                */
  float clip_norm;       /* > 0: clip the global gradient norm to this value       *
                          * (coef = min(1, clip / (||g|| + 1e-6)), the formula of  *
                          * torch clip_grad_norm_; R28).  0 = off.       */
  int skip_nonfinite;    /* 1: a step whose reduced gradient has an inf/NaN leaves *
                          * master, m, v and the parameters unchanged.  0 = flag   *
                          * only (default).  clip_norm > 0 or skip_nonfinite = 1   *
                          * selects the two-phase step: every bucket is reduced    *
                          * and the norm all-reduced before the first update, and  *
                          * the reduced gradient stays resident (psi/div(OS) bf16) */
  int fuse_gather;       /* when the parameter restore is one ring (AG_E for P = I,*
                          * OS = G; AG_I for P = N, OS = I; the world ring when    *
                          * M = 1 or g = 1) the Adam kernel can store its bf16     *
                          * output straight into the consumers' buffers over       *
                          * NVLink instead of a separate all-gather launch (same   *
                          * bits, same bytes per link class).  1 (default): only   *
                          * when no collective rounds run beside Adam (the whole   *
                          * reduction fused too); 2: always; 0: never.             */
  int copy_engine;       /* 1: collective launches that only copy bits (parameter  *
                          * all-gathers) run on the copy engines: per round a peer *
                          * barrier, then cudaMemcpyAsync over NVLink (bidirectional *
                          * ring traffic measured 770 GB/s/dir for the copy engines *
                          * vs 660 for SM loads, profiles/r01/p2p_bidir.jsonl);     *
                          * 2: also G = I's intra reduce-scatter as copy-engine     *
                          * copies of the peers' raw chunks + one local fold.       *
                          * 3: 1, and the trailing copy-only rounds of a reduce    *
                          * launch (the all-gather half of an all-reduce: OS = N,  *
                          * or AG_E for G = N, OS = I) leave the rounds kernel for *
                          * the copy engines, on a second stream: the kernels of   *
                          * later buckets run beside them (real mode only).        *
                          * 0 (default): the rounds kernel.  Measured in the full  *
                          * 7B IIG step at 2x2 (profiles/r02/                      *
                          * sweep_copy_engine_iig_2x2.jsonl): 0 / 1 / 2 = 21.10 /  *
                          * 20.43 / 20.49 ms; bench.py runs 1.                     */
  int gather_windows;    /* > 0: that many library window slots of bucket_elems    *
                          * bf16 each for paro_gather_window (P = I or G only).    */
  int grad_accum;        /* 1: enable paro_accumulate (gradient accumulation over  *
                          * s > 1 micro-batches); G = N plans then own  *
                          * a psi_pad bf16 accumulator.  0 (default): off.         */
  void* stream;          /* cudaStream_t the step is ordered on; NULL = ctx stream */
  int frozen;            /* 1: a frozen-parameter plan (partial / PEFT training:  *
                          * Psi' < Psi trainable; the frozen tensors keep  *
                          * only their parameters, 2 bytes each).  It owns *
                          * the P residency of its tensors and serves            *
                          * paro_gather_window; paro_step, paro_accumulate,       *
                          * paro_synth_grads and paro_collective return           *
                          * PARO_ERR_STATE; paro_opt_state_init* take st = NULL   *
                          * and only fill the parameter buffer.  Pair it with a   *
                          * plan of the trainable tensors (paro_plan_masked).    *
                          * 0 (default).                                          */
  int grad_slots;        /* K > 0: streamed gradients.  Instead of one psi_pad     *
                          * flat gradient buffer (2 Psi bytes, which Table 2 does  *
                          * not count for G = I / G), the plan keeps K bucket      *
                          * slots (2 K B bytes) and paro_step_streamed has each    *
                          * bucket's gradients produced into slot b % K just       *
                          * before its reduction, so a rank's memory is Table 2's  *
                          * P + G + OS plus staging.  paro_step and                *
                          * paro_synth_grads then return PARO_ERR_STATE; not with  *
                          * grad_accum; copy_engine is forced to 0.  0 (default).  */
  int fuse_allreduce;    /* OS = I with g = 2 groups (NII, III, INI, NNI,  *
                          * P:355 "all-reduce among groups"): 1 (default) folds    *
                          * the inter-group all-reduce AR_E into the Adam kernel,  *
                          * which reads the same-position peer's intra partial    *
                          * over NVLink beside its own (R31: at g = 2 the fold     *
                          * R_2 of both segments is one commutative bf16 add, so   *
                          * the bits equal the RS_E + AG_E ring; bytes per link    *
                          * class are equal too: (g-1)/g * 2 B/M = B/M).  G = I:  *
                          * the G residency then keeps the intra partial (R26);   *
                          * G = N: RS_I lands in the g_hat slot.  M = 1 (2 x 1):   *
                          * every OS != G code, the partials being the raw         *
                          * gradients.  Topologies HO, two-step, direct (any for   *
                          * G = I except NCCL).  Off with pull_transport = 0,      *
                          * clipping / skip and inter_gbps pacing.  0: the ring,   *
                          * and no part of any reduction runs inside Adam (the     *
                          * OS = G final hop stays in the rounds kernel too), so   *
                          * paro_collective(0) performs the whole reduction.       */
  int adam_smem_kb;      /* > 0: shared memory (KB) the TMA Adam kernel may use for *
                          * its stages, overriding the automatic 200 KB alone /    *
                          * ~120 KB beside collectives (so an emulated or N = 1    *
                          * run executes the co-run variants: 4096- or 2048-elem   *
                          * tiles, 2-4 stages).  0 (default): automatic.  Must be  *
                          * <= 220.                                                 */
  int wire_dtype;        /* 0 (default): bf16 wire (G is 2 bytes): every hop *
                          * RNE_bf16(fp32 a + fp32 b), g_hat bf16.  1: fp32 wire   *
                          * (reading A3): pre-scaled raw gradients, partials, the  *
                          * G residency and g_hat are fp32 (4 B per element on the *
                          * wire and in those buffers; bytes sent double), every   *
                          * hop one fp32 add, g_hat never rounded to bf16, so the  *
                          * result depends on the split / bucket only through fp32 *
                          * summation order (<= 1e-5 after 10 steps, SURVEY        *
                          * §8(c-4)); gradient accumulators are fp32 too.  Not     *
                          * with copy_engine = 2.                                  */
  int predivide;         /* 1 (default): raw gradients are multiplied by 1/N when   *
                          * first read (R4); 0: the raw sum is reduced and the 1/N *
                          * average is applied in Adam's unscale, s_g = 1 /        *
                          * (loss_scale * N) (reading A4; same bits for N = 2^k).  */
  const int64_t* bucket_groups; /* layer-aligned buckets (NEXT-2): n     *
                          * ascending tensor indices, the first 0; bucket k holds *
                          * exactly tensors [bucket_groups[k], bucket_groups[k+1]) *
                          * (dense, zero-padded at its end to a multiple of N*64), *
                          * so paro_gather_window(b) returns one layer group and a *
                          * caller can prefetch group b+1 while computing group b. *
                          * bucket_elems is then ignored; the flat layout has     *
                          * padding inside (paro_bucket_range, and per-tensor     *
                          * offsets follow the groups).  Read during paro_plan    *
                          * only.  NULL / 0 (default): dense layout, fixed buckets. */
  int n_bucket_groups;
} paro_opts_t;

typedef struct {
  int64_t psi;           /* sum of param sizes                              */
  int64_t psi_pad;       /* psi rounded up to a multiple of N*64 (R21)              */
  int64_t bucket_elems;  /* effective bucket size B                                 */
  int64_t n_buckets;
  int64_t p_numel, g_numel, os_numel;  /* per-rank residency sizes (elements)      */
  int64_t mem_p_bytes, mem_g_bytes, mem_os_bytes;  /* Table 2 at psi_pad           */
  int64_t workspace_bytes;             /* library staging per rank                 */
  int64_t step_send_bytes_intra;       /* this rank, one step, counted from the    */
  int64_t step_send_bytes_inter;       /*   transfers the kernels perform          */
  int32_t n_rounds;                    /* collective rounds per step (all buckets) */
  int32_t n_comm_launches;             /* collective kernel launches per step      */
  /* grad_accum plans: this rank's bytes per paro_accumulate call, and per      *
   * paro_step that follows accumulation (0 otherwise)                         */
  int64_t accum_send_bytes_intra, accum_send_bytes_inter;
  int64_t accum_step_send_bytes_intra, accum_step_send_bytes_inter;
  int64_t grad_buffer_bytes;           /* raw gradient buffer per rank: 2 psi_pad, or *
                                        * 2 K B with grad_slots = K                    */
} paro_plan_info_t;

typedef struct {
  double grad_norm;      /* sqrt(sum (g_hat * s_g)^2) over unique elements (R8)     */
  int32_t nonfinite;     /* 1 if any reduced gradient was inf/NaN (R9: flag only)   */
  int64_t sent_intra, sent_inter;  /* bytes this rank sent in the last step         */
  int32_t kernel_launches;         /* library kernels launched by the last step     */
  /* NVLink bytes this rank's transfers moved since the last paro_step began, by  *
   * link class: counted on the device by the kernels that move them (every tile *
   * a CTA pulls from a peer or pushes into one; fused-hop pulls and fused-gather *
   * pushes in Adam), plus copy-engine copies counted at enqueue.  In these       *
   * rank-symmetric schedules it equals sent_intra / sent_inter (except H-Ring,   *
   * whose leaders pull more than they are pulled: totals over ranks agree).      *
   * Real mode only; -1 in emulated mode and for the NCCL comparator.             */
  int64_t moved_intra, moved_inter;
} paro_step_stats_t;

/* Fill *o with the defaults listed above. */
void paro_opts_default(paro_opts_t* o);

/* ---- contexts ------------------------------------------------------------ */

/* New NCCL unique id; call on rank 0 and broadcast (e.g. with torch.distributed). */
paro_status_t paro_get_unique_id(paro_uid_t* out);

/* One rank of a real N-GPU job (one process per GPU).  world_size = N,
 * group_size = M must divide N ("group_size must divide n_gpus").
 * Creates the NCCL world communicator from uid, its intra (color = group) and
 * inter (color = position) splits, the streams, and maps peer memory.
 * Collective: all ranks must call it. */
paro_status_t paro_init(int world_size, int group_size, int rank, const paro_uid_t* uid,
                        int device, paro_ctx_t* out);

/* All N ranks emulated in this one process on one device (no NCCL, no peer
 * memory): every collective round becomes one kernel over all ranks' data.
 * Used for bit-exact tests of any split on one GPU. */
paro_status_t paro_init_emulated(int world_size, int group_size, int device, paro_ctx_t* out);

/* Planning-only context: no CUDA calls.  paro_plan / paro_plan_info /
 * paro_shard_range / paro_rank_send_bytes work; buffers and steps do not. */
paro_status_t paro_init_planner(int world_size, int group_size, paro_ctx_t* out);

paro_status_t paro_finalize(paro_ctx_t ctx);

/* ---- plans ------------------------------------------------------------------ */

/* Validate `strategy` (3 letters over {N,I,G} in P/G/OS order, Table 1; error
 * strings "invalid shard level 'X' at position k", "strategy 'GGN' violates
 * Principle 1 (S_P>=S_OS and S_G>=S_OS)"), lay the n_params tensors of
 * param_sizes out densely in the given order, cut buckets, build the
 * position-major shard map (R1), the per-bucket collective schedule and the
 * accounting, and allocate the plan's device buffers (flat gradient buffer,
 * parameter buffer, G-residency buffer, staging).  Collective in real mode. */
paro_status_t paro_plan(paro_ctx_t ctx, const char* strategy, const int64_t* param_sizes,
                        int n_params, const paro_opts_t* opts, paro_plan_t* out);

/* Partial / PEFT training ("full, partial, and PEFT"; P:172 Psi' trainable
 * parameters; P:225 memory 2Psi, 2Psi', 12Psi'): trainable[i] != 0 marks tensor
 * i trainable.  Creates *out_trainable = paro_plan over the trainable tensors
 * (in their declaration order; the sync + update step runs on Psi' elements)
 * and *out_frozen = a frozen-parameter plan (opts->frozen = 1) over the others
 * (NULL when every tensor is trainable).  Both use `strategy`'s P level, so
 * every parameter is resident at P and gathered the same way; G and OS exist
 * for the trainable tensors only.  Collective in real mode.  Errors as
 * paro_plan; PARO_ERR_INVALID if no tensor is trainable. */
paro_status_t paro_plan_masked(paro_ctx_t ctx, const char* strategy, const int64_t* param_sizes,
                               const uint8_t* trainable, int n_params, const paro_opts_t* opts,
                               paro_plan_t* out_trainable, paro_plan_t* out_frozen);

paro_status_t paro_plan_info(paro_plan_t plan, paro_plan_info_t* out);

/* Flat element range [*begin, *end) of state (0 = P, 1 = G, 2 = OS) held by
 * `rank` inside bucket `bucket` (position-major nested map, R1). */
paro_status_t paro_shard_range(paro_plan_t plan, int state, int rank, int64_t bucket,
                               int64_t* begin, int64_t* end);

/* Bucket [*begin, *end) in the flat parameter space. */
paro_status_t paro_bucket_range(paro_plan_t plan, int64_t bucket, int64_t* begin, int64_t* end);

/* Bytes `rank` sends per step on intra- and inter-group links, counted from the
 * plan's transfer list (pull model, a byte read by a peer from this
 * rank's memory counts as sent by this rank). */
paro_status_t paro_rank_send_bytes(paro_plan_t plan, int rank, int64_t* intra, int64_t* inter);

/* grad_accum plans: bytes `rank` sends per paro_accumulate call (*acc_*) and
 * in the paro_step that follows accumulation (*step_*), per link class,
 * counted from the transfer lists like paro_rank_send_bytes.  PARO_ERR_STATE
 * if the plan was made with grad_accum = 0. */
paro_status_t paro_rank_accum_send_bytes(paro_plan_t plan, int rank, int64_t* acc_intra, int64_t* acc_inter,
                                         int64_t* step_intra, int64_t* step_inter);

/* Forward / backward parameter all-gather ("model parameters are
 * ... intra-group sharded"; "each GPU obtains a complete replica of
 * model parameters through the intra-group all-gather operation", P:341;
 * Table 3 columns Forward / Backward A-G(P)).  Assembles bucket `bucket`'s
 * full bf16 parameters (flat layout of paro_bucket_range) of local `rank`
 * into window slot `slot` and returns its device address in *out: P = I
 * gathers inside the group (ring AG_I), P = G over all ranks on the plan's
 * topology (HO-Ring by default).  Bit copies: the window equals the bucket
 * slice of the full model's bf16 parameters after the last step.
 * Stream-ordered on `stream` (NULL = the plan stream), so a caller can
 * prefetch bucket b+1 on a side stream while computing on bucket b; the
 * window may be reused once the caller's reads of it are stream-ordered
 * before the next gather into the same slot.  Collective over the ranks the
 * level spans.  P = N (or N = 1): no transfer, *out points into the
 * parameter buffer.  Emulated mode: rank 0, all ranks gather at once.
 * Errors: PARO_ERR_STATE if the plan has no windows (gather_windows = 0). */
paro_status_t paro_gather_window(paro_plan_t plan, int rank, int64_t bucket, int slot, void* stream, void** out);

/* Bytes `rank` sends to gather every bucket once through paro_gather_window. */
paro_status_t paro_rank_gather_send_bytes(paro_plan_t plan, int rank, int64_t* intra, int64_t* inter);

/* Bytes `rank` sends in one paro_gather_window of bucket `bucket` (with
 * bucket_groups: one layer group's forward or backward A-G(P), Table 3). */
paro_status_t paro_bucket_gather_send_bytes(paro_plan_t plan, int rank, int64_t bucket, int64_t* intra,
                                            int64_t* inter);

/* Library-owned device buffers of `rank` (must be a local rank):
 *   kind 0: flat gradient buffer, bf16, psi_pad elements (zero-padded tail).
 *           Writing gradients here and passing grads = NULL to paro_step is
 *           the zero-copy path.
 *   kind 1: parameter buffer, bf16, p_numel elements (P residency, bucket-major).
 *   kind 2: G-residency buffer, bf16 (fp32 on the fp32 wire), g_numel elements
 *           (NULL for G = N, whose gradient residency is the flat gradient buffer).
 *   kind 3: reduced-gradient slots (bf16, fp32 on the fp32 wire; slot b % (pipeline_depth+1) holds
 *           bucket b's g_hat at the OS residency) or NULL when g_hat lives in
 *           the G-residency buffer or is consumed directly by Adam.
 *   kind 4: the G = N gradient accumulator (bf16, psi_pad elements; grad_accum
 *           plans with G = N only, else NULL).
 *   kind 5: parameter-gather window slot 0 (gather_windows x bucket_elems bf16,
 *           slot w at + 2 * w * bucket_elems bytes; NULL without windows). */
paro_status_t paro_buffer(paro_plan_t plan, int rank, int kind, void** ptr);

/* Initialise one local rank's optimizer state and parameter buffer from a full
 * fp32 master vector `master_full` (device, psi_pad elements in the plan's flat
 * layout: param i at its flat offset, padding ignored; for the dense layout
 * the first psi elements suffice):
 * master = its OS residency slice, m = v = 0, param buffer = RNE_bf16 of the P
 * residency slice.  Stream-ordered on the plan stream. */
paro_status_t paro_opt_state_init(paro_plan_t plan, int rank, const float* master_full,
                                  const paro_opt_state_t* st);

/* Same, with master weights from the counter-based synthetic generator
 * (paro_synth) instead of a vector: no psi-sized temporary. */
paro_status_t paro_opt_state_init_synth(paro_plan_t plan, int rank, uint64_t seed,
                                        const paro_opt_state_t* st);

/* Fill a local rank's flat gradient buffer with synthetic bf16 gradients of
 * (seed, rank, step). */
paro_status_t paro_synth_grads(paro_plan_t plan, int rank, uint64_t seed, int64_t step);

/* One s = 1 sync + update step, stream-ordered and asynchronous.
 *  grads:  NULL = gradients already in each local rank's flat gradient buffer;
 *          else n_params bf16 device pointers per local rank (rank-major in
 *          emulated mode), packed into the flat buffer first.
 *  params: NULL = the plan's parameter buffer is the destination (zero copy);
 *          else per local rank: n_params bf16 pointers (P = N) or one pointer
 *          to p_numel elements (P = I, G) that receive a copy after the step.
 *  opt_state: one paro_opt_state_t per local rank (rank order).
 *  lr: this step's learning rate; step: 1-based Adam t ("step must be >= 1").
 *  After paro_accumulate calls, grads must be NULL: the step consumes the
 *  accumulator ("grads must be NULL after paro_accumulate"). */
paro_status_t paro_step(paro_plan_t plan, const void* const* grads, void* const* params,
                        const paro_opt_state_t* opt_state, float lr, int64_t step);

/* Streamed step (plans with grad_slots = K > 0): the same step as paro_step,
 * but bucket b's raw gradients are written into slot b % K while the step runs
 * (ZeRO-style bucketed gradients: a rank never holds all of them, P:343-344,
 * Table 2's G column).  For every bucket in order and every local rank, once
 * every rank is done reading bucket b - K from that slot, the library calls
 *   producer(user, rank, b, begin, end, dst, stream)
 * from this host thread; it must enqueue, on `stream` (a cudaStream_t), writes
 * of the bf16 gradients of flat elements [begin, end) (paro_bucket_range;
 * zero on padding) into the device buffer dst (end - begin elements), and
 * return.  producer NULL: the library's synthetic gradients of `seed` and
 * `grad_step` (the paro_synth_grads values).  params, opt_state, lr, step:
 * as paro_step.  Errors: PARO_ERR_STATE if the plan has no grad_slots. */
typedef void (*paro_grad_producer_t)(void* user, int rank, int64_t bucket, int64_t begin, int64_t end,
                                     void* dst, void* stream);
paro_status_t paro_step_streamed(paro_plan_t plan, paro_grad_producer_t producer, void* user, uint64_t seed,
                                 int64_t grad_step, void* const* params, const paro_opt_state_t* opt_state,
                                 float lr, int64_t step);

/* Parameter consumer: after paro_set_param_consumer, every paro_step /
 * paro_step_streamed calls, for each bucket b in order and every local rank,
 *   consumer(user, rank, b, begin, end, src, stream)
 * from the calling host thread; it must enqueue, on `stream` (a cudaStream_t
 * that waits until bucket b's updated bf16 parameters are final on this rank:
 * after its restore, or its Adam when there is none, and with fused gathers
 * after every peer's Adam of b), reads of the rank's P residency of the bucket:
 * flat elements [begin, end) (paro_shard_range(P)), `end - begin` bf16 at src.
 * The step completes (on its stream) only once these reads have.  Use: copy
 * each bucket device->host while later buckets still reduce / update (and, in
 * a streamed step, while their gradients come in: PCIe is full duplex).
 * consumer NULL unregisters.  Errors: PARO_ERR_STATE on a planning-only
 * context or a frozen-parameter plan. */
typedef void (*paro_param_consumer_t)(void* user, int rank, int64_t bucket, int64_t begin, int64_t end,
                                      const void* src, void* stream);
paro_status_t paro_set_param_consumer(paro_plan_t plan, paro_param_consumer_t consumer, void* user);

/* Gradient accumulation (§3.3; R27).  Adds one
 * micro-batch's gradients at the G residency: G = G reduces the micro-batch
 * over all ranks (HO-Ring RS), G = I inside the group (RS_I, P:353,
 * P:369), G = N only locally; the result is folded into the rank's bf16
 * accumulator, acc = acc (+) r (first call: acc = r).  After s >= 1 calls the
 * next paro_step (grads must be NULL) finishes the reduction from the
 * accumulator once (G = I: the inter-group RS / AR, "only once"), runs
 * Adam on the mini-batch mean (unscale 1/(loss_scale * s)) and the parameter
 * all-gather, and resets s.  Per-rank bytes: paro_plan_info_t.accum_*.
 *  grads: NULL = the micro-batch is in each local rank's flat gradient buffer
 *         (paro_buffer kind 0); else n_params bf16 device pointers per local
 *         rank, packed first.  The gradient buffer may be overwritten once the
 *         call's work has completed on the stream.
 * Errors: PARO_ERR_STATE if the plan was made with grad_accum = 0. */
paro_status_t paro_accumulate(paro_plan_t plan, const void* const* grads);

/* Collective only (no optimizer): run the plan's gradient-reduction launches
 * (what = 0) or parameter all-gather launches (what = 1) for every bucket,
 * stream-ordered like paro_step.  With strategy NNN and fuse_allreduce = 0,
 * what = 0 is a hierarchical all-reduce of the flat gradient buffer
 * (gradients pre-scaled by 1/N, i.e. the average) on the plan's topology: the
 * HO-Ring all-reduce of BASELINE config 5 (bucket b's average lands in
 * paro_buffer kind 3, slot b % (pipeline_depth + 1)).
 * Requires a real or emulated context.  PARO_ERR_STATE for what = 0 on a plan
 * that folds part of its reduction into the Adam kernel (fuse_allreduce = 1:
 * the inter all-reduce at g = 2, or the final hop of OS = G): its reduce
 * launches alone do not complete the reduction. */
paro_status_t paro_collective(paro_plan_t plan, int what);

/* Per-kernel timing over a region of steps (used by bench.py for the roofline):
 * paro_profile_start allocates `max_launches` CUDA event pairs and brackets
 * every following library kernel launch on the stream it runs on;
 * paro_profile_stop synchronises, sums the per-launch durations by kind and
 * stops recording.  Launches beyond max_launches are not timed. */
typedef struct {
  double adam_ms;        /* sum of fused-Adam kernel durations                    */
  double comm_ms;        /* sum of collective (rounds / NCCL) launch durations    */
  int64_t adam_launches, comm_launches;
  int64_t adam_elems;    /* elements the timed Adam launches processed            */
  int64_t comm_bytes;    /* bytes this rank sent in the timed collective launches */
  int64_t steps;         /* paro_step calls inside the region                     */
  int64_t kernel_launches; /* all library kernel launches inside the region       */
  /* device-side globaltimer trace of the first (up to 512) collective launches
   * of the region (real mode): time in peer/grid barriers before each round,
   * in the rounds' data movement, and in the launch-final barrier */
  int64_t traced_launches;
  double traced_barrier_ms, traced_work_ms, traced_final_ms;
  /* algorithmic HBM bytes of this GPU in the timed launches: Adam = 26 B +
   * 2 B per g_hat input (fused final hop) + 2 B per fused-gather push, per
   * element; collectives = 2 B per task input + 2 B per output element */
  int64_t adam_hbm_bytes, comm_hbm_bytes;
  /* the last Adam launch: 0 adam_kernel (LSU), 1 adam_tma_kernel<false,512>   *
   * (bulk loads, thread stores), 2 <true,512> (bulk loads + stores), 3       *
   * <true,256>, 4 <false,256>, 5 adam_tma_ws_kernel<512> (warp-specialized),  *
   * 6 adam_tma_ws_kernel<256>; -1 none; and its shared-memory stage count     */
  int32_t adam_variant, adam_stages;
} paro_profile_t;

paro_status_t paro_profile_start(paro_plan_t plan, int max_launches);
paro_status_t paro_profile_stop(paro_plan_t plan, paro_profile_t* out);

/* Synchronise the plan stream and return the last step's statistics.
 * Returns PARO_ERR_TIMEOUT if a cross-GPU wait timed out on the device. */
paro_status_t paro_step_stats(paro_plan_t plan, paro_step_stats_t* out);

paro_status_t paro_plan_destroy(paro_plan_t plan);

/* Thread-local message of the last failed call on this thread. */
const char* paro_last_error(void);

/* Library version string ("paro-b200 <semver> sm_100a"). */
const char* paro_version(void);

/* ---- strategy advisor (NEXT-4; reading R29) ----------------------
 * Table 1 marks the codes recommended for each training type;
 * §3.1 trades memory (Table 2; P, G, OS take 2Psi, 2Psi',
 * 12Psi' bytes) against communication (Table 3).  paro_advise evaluates all 14
 * strategies for one task and returns them ranked: recommended-and-fitting
 * first, then by modeled communication time, memory, code. */
typedef struct {
  int n_gpus, group_size;     /* N and M (M divides N)                                 */
  int64_t psi;                /* model parameters Psi                           */
  int64_t psi_trainable;      /* trainable parameters Psi' (0 < Psi' <= Psi)     */
  int accum_steps;            /* s micro-batches per mini-batch, >= 1           */
  int peft;                   /* 1: PEFT task (Table 1's last column, Psi' << Psi)      */
  double mem_budget_bytes;    /* model-state bytes available per GPU                    */
  double bw_intra_gbs;        /* per-rank intra-group link bandwidth, GB/s              */
  double bw_inter_gbs;        /* per-rank inter-group link bandwidth, GB/s              */
} paro_advise_in_t;

typedef struct {
  char code[4];               /* "IIG", NUL-terminated                                  */
  int32_t recommended;        /* Table 1 mark in the task's column                      */
  int32_t fits;               /* mem_bytes <= mem_budget_bytes                          */
  int64_t mem_bytes;          /* 2Psi/div(P) + 2Psi'/div(G) + 12Psi'/div(OS), padded R21 */
  int64_t intra_bytes;        /* bytes the busiest rank sends per mini-batch: s x       */
  int64_t inter_bytes;        /*   (fwd + bwd param gather + micro-batch reduction) +   *
                               *   the update-stage ops, counted from the library's own *
                               *   plans (HO-Ring topology)                             */
  double t_comm_s;            /* intra / bw_intra + inter / bw_inter                    */
} paro_advice_t;

/* Table 1 column of a task: 0 Psi' = Psi, 1 Psi' >= Psi/6, 2 Psi' < Psi/6, 3 PEFT. */
int paro_table1_column(int64_t psi, int64_t psi_trainable, int peft);

/* Fill out[0..13] (cap >= 14) with every PaRO strategy, best first; *n_out = 14.
 * Host only (no context needed).  PARO_ERR_INVALID on a bad cluster shape,
 * sizes, accum_steps < 1 or non-positive bandwidths. */
paro_status_t paro_advise(const paro_advise_in_t* in, paro_advice_t* out, int cap, int* n_out);

#ifdef __cplusplus
}
#endif
#endif /* PARO_H_ */
