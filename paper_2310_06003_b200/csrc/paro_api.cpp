// paro_api.cpp — C ABI (include/paro.h) and the step engine.
//
// Engine per step (real or emulated mode), bucket b in order:
//   comm stream:    reduce(b)            [rounds kernel; NVLink pull + hop]
//   compute stream: adam(b)              [after reduce(b): fused Adam + bf16 cast]
//   comm stream:    gather(b - D)        [after adam(b - D): in-place all-gather]
// then the remaining gathers, the norm finalize (+ NCCL scalar all-reduce) and
// the join back onto the caller's stream.  Every rank issues the same launch
// sequence, so the in-kernel peer barriers pair up.
#include <cuda_runtime.h>
#include <nccl.h>

#include <nvtx3/nvToolsExt.h>

#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/paro.h"
#include "kernels.h"
#include "planner.h"

using namespace paro;

namespace {

thread_local std::string g_last_error;

paro_status_t fail(paro_status_t st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

enum Mode { MODE_REAL = 0, MODE_EMU = 1, MODE_PLANNER = 2 };

}  // namespace

namespace paro {
paro_status_t api_fail(paro_status_t st, const std::string& msg) { return fail(st, msg); }
}  // namespace paro

struct paro_ctx {
  int mode = MODE_PLANNER;
  int N = 1, M = 1, rank = 0, device = -1;
  cudaStream_t main = nullptr, comm = nullptr, comp = nullptr;
  cudaStream_t dma = nullptr;   // copy-engine transfers of pure-copy launches
  cudaStream_t sink = nullptr;  // parameter consumer (paro_set_param_consumer): per-bucket reads
  ncclComm_t world = nullptr, intra = nullptr, inter = nullptr;
  paro_status_t sticky = PARO_OK;
  std::string sticky_msg;
  int sm_count = 148;
};

struct CopyOp {
  void* dst;
  const void* src;
  size_t bytes;
};

struct DevLaunch {
  // pure-copy launch run by the copy engines (opts.copy_engine): per round a
  // 1-CTA barrier kernel on the second barrier channel, then cudaMemcpyAsync
  bool dma = false;
  std::vector<std::vector<CopyOp>> copies;   // [round] local rank(s)' copies
  std::vector<uint64_t> round_peers;         // [round] barrier peers before it
  int max_in = 1;          // largest fold input count (TMA stage sizing)
  int generic = 0;         // has fp32-wire or nested (one-shot) tasks: the generic fold kernel
  int64_t bytes = 0;       // bytes the local rank(s) send in this launch
  int64_t hbm = 0;         // algorithmic HBM bytes of the local rank(s)' tasks: each input
                           // read once (a peer's input is read from its HBM; by symmetry
                           // the same bytes a peer reads here) + the output written
  int64_t round_off = 0;   // index into the plan's DRound array
  int nrounds = 0;
  int final_barrier = 0;
  uint64_t final_peers = 0;
  // copy-engine tail (opts.copy_engine = 3): the launch's trailing pure-copy
  // rounds, run by the copy engines after the kernel's rounds [0, nrounds)
  std::vector<DevLaunch> tail;
};

struct paro_plan {
  paro_ctx* ctx = nullptr;
  std::unique_ptr<Planner> pl;
  paro_opts_t opts{};
  std::vector<int> local;                 // local ranks (real: {rank}, emulated: all)
  std::vector<char*> region;              // per local rank: device region base
  std::vector<char*> peer_base;           // [N] base as addressable from this process
  uint64_t** d_peer_slot = nullptr;       // real mode
  uint64_t** d_peer_slot2 = nullptr;      // second barrier channel (copy-engine launches)
  uint64_t** d_peer_slot3 = nullptr;      // third channel (parameter consumer stream)
  paro_param_consumer_t cons_fn = nullptr;  // per-bucket consumer of the updated parameters
  void* cons_user = nullptr;
  cudaEvent_t ev_cons = nullptr;
  std::vector<cudaEvent_t> ev_pfinal;     // bucket b's parameters final on this rank
  cudaEvent_t ev_dma = nullptr;
  cudaEvent_t ev_tail = nullptr;          // comm -> dma hand-over of a copy-engine tail
  DRound* d_rounds = nullptr;
  DTask* d_tasks = nullptr;
  std::vector<DevLaunch> red, gat;        // per bucket
  std::vector<DevLaunch> acc_first, acc_next, red_acc;   // gradient accumulation (per bucket)
  std::vector<std::vector<DevLaunch>> win;  // [window slot][bucket]: forward/backward parameter gather
  std::vector<DevLaunch> red_pre, acc_pre;  // copy-engine raw-chunk copies before reduce / accum (per bucket)
  std::vector<cudaEvent_t> ev_pre;
  std::vector<cudaEvent_t> ev_prod;       // streamed step: bucket b's gradients are in their slot
  int64_t acc_count = 0;                  // micro-batches accumulated since the last step
  bool last_step_acc = false;             // the last step consumed an accumulator
  double* d_partials = nullptr;
  int partials_cap = 0;
  double* d_norm = nullptr;
  int* d_nonfinite = nullptr;
  float* d_sg = nullptr;                  // two-phase step: device unscale factor (clip)
  int* d_skip = nullptr;                  // two-phase step: skip the update
  PackEntry* d_pack = nullptr;
  PackEntry* h_pack = nullptr;            // pinned staging
  int pack_cap = 0;
  cudaEvent_t ev_fork = nullptr, ev_comm = nullptr, ev_comp = nullptr, ev_pack_staged = nullptr,
              ev_unpack_staged = nullptr;
  std::vector<cudaEvent_t> ev_red, ev_adam;
  cudaStream_t last_stream = nullptr;
  int last_launches = 0;
  bool stepped = false;
  // profiling (paro_profile_start / stop)
  bool prof = false;
  std::vector<cudaEvent_t> prof_ev;       // 2 per launch
  std::vector<int> prof_kind;             // 0 adam, 1 comm
  std::vector<int64_t> prof_amount;       // adam: elements; comm: bytes sent
  std::vector<int64_t> prof_hbm;          // algorithmic HBM bytes of the launch (this GPU)
  int prof_used = 0;
  int64_t prof_steps = 0, prof_launches = 0;
  int adam_variant = -1, adam_stages = 0;   // the last Adam launch (AdamVariant)
  unsigned long long* d_moved = nullptr;    // [intra, inter] NVLink bytes moved by this rank's kernels
  int64_t moved_host[2] = {0, 0};           // ... by its copy-engine transfers (counted at enqueue)
  float alpha = 1.f;                        // pre-scaling of raw gradients: 1/N (predivide) or 1
  uint64_t* d_trace = nullptr;            // [kTraceLaunches][grid][kTraceSlots]
  std::vector<int> trace_nrounds;         // rounds of each traced launch
  std::vector<int> trace_grids;           // CTAs of each traced launch (stride: sm_count)
};
// (the C API also declares a *function* named paro_plan, which hides the tag in C++)
using PlanT = struct paro_plan;

namespace {

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) return cuda_fail(ctx, #call, e_);                             \
  } while (0)
#define NK(call)                                                                         \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess) return nccl_fail(ctx, #call, r_);                             \
  } while (0)

paro_status_t cuda_fail(paro_ctx* ctx, const char* what, cudaError_t e) {
  std::string m = std::string(what) + ": " + cudaGetErrorString(e);
  if (ctx) {
    ctx->sticky = (e == cudaErrorMemoryAllocation) ? PARO_ERR_OOM : PARO_ERR_CUDA;
    ctx->sticky_msg = m;
    if (e == cudaErrorMemoryAllocation) ctx->sticky = PARO_OK;  // OOM is not sticky
    return fail(e == cudaErrorMemoryAllocation ? PARO_ERR_OOM : PARO_ERR_CUDA, m);
  }
  return fail(PARO_ERR_CUDA, m);
}

paro_status_t nccl_fail(paro_ctx* ctx, const char* what, ncclResult_t r) {
  std::string m = std::string(what) + ": " + ncclGetErrorString(r);
  if (ctx) {
    ctx->sticky = PARO_ERR_NCCL;
    ctx->sticky_msg = m;
  }
  return fail(PARO_ERR_NCCL, m);
}

// Synchronise `s` while polling the NCCL communicators' asynchronous error
// state (a failed or aborted peer surfaces here instead of a silent hang);
// after PARO_WATCH_S seconds (default 300) without completion the context is
// marked timed out.  The in-kernel peer waits time out on their own (20 s).
paro_status_t sync_watch(paro_ctx* ctx, cudaStream_t s) {
  const double limit = std::getenv("PARO_WATCH_S") ? std::atof(std::getenv("PARO_WATCH_S")) : 300.0;
  const auto t0 = std::chrono::steady_clock::now();
  for (int it = 0;; ++it) {
    cudaError_t q = cudaStreamQuery(s);
    if (q == cudaSuccess) return PARO_OK;
    if (q != cudaErrorNotReady) return cuda_fail(ctx, "cudaStreamQuery", q);
    for (ncclComm_t c : {ctx->world, ctx->intra, ctx->inter}) {
      if (!c) continue;
      ncclResult_t ae = ncclSuccess;
      ncclResult_t r = ncclCommGetAsyncError(c, &ae);
      if (r != ncclSuccess) return nccl_fail(ctx, "ncclCommGetAsyncError", r);
      if (ae != ncclSuccess && ae != ncclInProgress) return nccl_fail(ctx, "NCCL asynchronous error", ae);
    }
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > limit) {
      ctx->sticky = PARO_ERR_TIMEOUT;
      ctx->sticky_msg = "the step did not complete within PARO_WATCH_S seconds";
      return fail(PARO_ERR_TIMEOUT, ctx->sticky_msg);
    }
    std::this_thread::sleep_for(std::chrono::microseconds(it < 100 ? 20 : 500));
  }
}

paro_status_t check_ctx(paro_ctx* ctx) {
  if (!ctx) return fail(PARO_ERR_INVALID, "null context");
  if (ctx->sticky != PARO_OK) return fail(ctx->sticky, "sticky error: " + ctx->sticky_msg);
  if (ctx->mode != MODE_PLANNER) {
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return cuda_fail(ctx, "cudaSetDevice", e);
  }
  return PARO_OK;
}

// NVTX range over the host-side enqueue of a step / bucket launch (visible to
// Nsight tools when attached; a no-op otherwise, NVTX3 is header-only)
struct NvtxRange {
  explicit NvtxRange(const char* fmt, ...) {
    char buf[96];
    va_list ap;
    va_start(ap, fmt);
    std::vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    nvtxRangePushA(buf);
  }
  ~NvtxRange() { nvtxRangePop(); }
};

bool is_local(const PlanT* p, int rank) {
  for (int r : p->local)
    if (r == rank) return true;
  return false;
}

int local_index(const PlanT* p, int rank) {
  for (size_t i = 0; i < p->local.size(); ++i)
    if (p->local[i] == rank) return (int)i;
  return -1;
}

char* data_ptr(const PlanT* p, int rank, int kind, int64_t off) {
  const Planner& pl = *p->pl;
  return p->peer_base[rank] + kHeaderBytes + pl.buf_off[kind] + (int64_t)pl.esz[kind] * off;
}

// which rank's region a resolved device pointer belongs to (-1: none)
int data_rank(const PlanT* p, const void* ptr) {
  const char* c = static_cast<const char*>(ptr);
  const size_t bytes = kHeaderBytes + (size_t)p->pl->region_bytes;
  for (int r = 0; r < (int)p->peer_base.size(); ++r)
    if (p->peer_base[r] && c >= p->peer_base[r] && c < p->peer_base[r] + bytes) return r;
  return -1;
}

// acc_kind >= 0: a task writing that buffer kind also folds its old contents in
// as the last input (gradient accumulation: acc = acc (+) r, R27)
DTask resolve(const PlanT* p, const Task& t, int executing_rank, int acc_kind, int64_t win_shift = 0) {
  DTask d{};
  auto ptr_of = [&](const Ref& x) {
    return data_ptr(p, x.rank, x.kind, x.off + (x.kind == BUF_WIN ? win_shift : 0));
  };
  d.nin = t.nin;
  d.n8 = t.n / 8;
  d.nest = (int16_t)t.nest;
  d.nblk = (int16_t)t.nblk;
  d.rawmask = 0;
  d.inter = 0;
  d.f32mask = 0;
  const Planner& pl = *p->pl;
  d.out_f32 = pl.esz[t.dst.kind] == 4 ? 1 : 0;
  const int M = pl.M;
  for (int i = 0; i < t.nin; ++i) {
    d.in[i] = reinterpret_cast<const uint16_t*>(ptr_of(t.in[i]));
    if (t.in[i].is_raw()) d.rawmask |= 1u << i;
    else if (pl.esz[t.in[i].kind] == 4) d.f32mask |= 1u << i;
    if (t.in[i].rank / M != executing_rank / M) d.inter += 1;
  }
  for (int i = 0; i < t.nin; ++i)
    if (t.in[i].rank != executing_rank) {
      d.peermask |= 1u << i;
      if (t.in[i].rank / M != executing_rank / M) d.intermask |= 1u << i;
    }
  if (t.dst.rank != executing_rank) d.dst_peer = (t.dst.rank / M != executing_rank / M) ? 2 : 1;
  for (int i = 0; i < t.nin; ++i)
    if ((d.peermask >> i) & 1u) {
      const int b = (!t.in[i].is_raw() && pl.esz[t.in[i].kind] == 4) ? 4 : 2;
      if ((d.intermask >> i) & 1u) d.mv_inter += b;
      else d.mv_intra += b;
    }
  if (d.dst_peer) (d.dst_peer == 2 ? d.mv_inter : d.mv_intra) += pl.esz[t.dst.kind];
  d.dst = reinterpret_cast<uint16_t*>(ptr_of(t.dst));
  if (t.dst.rank / M != executing_rank / M) d.inter += 1;
  if (acc_kind >= 0 && t.dst.kind == acc_kind) {
    if (d.out_f32) d.f32mask |= 1u << d.nin;
    d.in[d.nin++] = d.dst;
    if (t.dst.rank / M != executing_rank / M) d.inter += 1;
  }
  return d;
}

// Build device round/task arrays for every bucket's launches.
paro_status_t upload_schedule(PlanT* p) {
  paro_ctx* ctx = p->ctx;
  const Planner& pl = *p->pl;
  std::vector<DRound> rounds;
  std::vector<DTask> tasks;
  auto build = [&](const Launch& L, int acc_kind, int64_t win_shift = 0, bool allow_tail = false) {
    DevLaunch dl;
    dl.round_off = (int64_t)rounds.size();
    if (L.empty()) return dl;
    const int R = (int)L.rounds.size();
    for (int r = 0; r < R; ++r) {
      DRound d{};
      d.t0 = (int32_t)tasks.size();
      d.units = 0;
      if (ctx->mode == MODE_REAL) {
        for (const Task& t : L.rounds[r][ctx->rank]) {
          tasks.push_back(resolve(p, t, ctx->rank, acc_kind, win_shift));
          d.units += t.n / 8;
        }
        d.peers_before = L.barrier_peers(r, ctx->rank);
      } else {
        for (int x = 0; x < pl.N; ++x)
          for (const Task& t : L.rounds[r][x]) {
            tasks.push_back(resolve(p, t, x, acc_kind, win_shift));
            d.units += t.n / 8;
          }
        d.peers_before = 0;
      }
      d.t1 = (int32_t)tasks.size();
      for (int ti = d.t0; ti < d.t1; ++ti) {
        dl.max_in = std::max(dl.max_in, (int)tasks[ti].nin);
        if (tasks[ti].out_f32 || tasks[ti].nest > 1) dl.generic = 1;
      }
      (void)acc_kind;
      rounds.push_back(d);
    }
    dl.nrounds = R;
    dl.final_barrier = L.final_barrier ? 1 : 0;
    // bytes sent by the local rank(s): what peers read from them in this launch
    std::vector<int64_t> bytes_r(R, 0), hbm_r(R, 0);
    for (int r = 0; r < R; ++r)
      for (int x = 0; x < pl.N; ++x)
        for (const Task& t : L.rounds[r][x]) {
          for (int i = 0; i < t.nin; ++i) {
            const int y = t.in[i].rank;
            if (y != x && (ctx->mode != MODE_REAL || y == ctx->rank)) bytes_r[r] += pl.esz[t.in[i].kind] * t.n;
          }
          if (t.dst.rank != x && (ctx->mode != MODE_REAL || x == ctx->rank)) bytes_r[r] += pl.esz[t.dst.kind] * t.n;
        }
    for (int r = 0; r < R; ++r)
      for (int x = 0; x < pl.N; ++x) {
        if (ctx->mode == MODE_REAL && x != ctx->rank) continue;
        for (const Task& t : L.rounds[r][x]) {
          hbm_r[r] += pl.esz[t.dst.kind] * t.n;
          for (int i = 0; i < t.nin; ++i) hbm_r[r] += pl.esz[t.in[i].kind] * t.n;
        }
      }
    for (int r = 0; r < R; ++r) {
      dl.bytes += bytes_r[r];
      dl.hbm += hbm_r[r];
    }
    dl.final_peers = (ctx->mode == MODE_REAL) ? L.barrier_peers(R, ctx->rank) : 0;
    // copy engines: every task of round r (of every rank: the decision is the
    // same on all ranks, their barrier channels stay in step) a plain 1-input bit copy
    auto pure_round = [&](int r) {
      bool ok = true;
      for (int x = 0; x < pl.N && ok; ++x)
        for (const Task& t : L.rounds[r][x])
          ok = ok && t.nin == 1 && !t.in[0].is_raw() && pl.esz[t.in[0].kind] == pl.esz[t.dst.kind];
      return ok;
    };
    bool pure = p->opts.copy_engine != 0 && R > 0;
    for (int r = 0; r < R && pure; ++r) pure = pure_round(r);
    // copy-engine tail (copy_engine = 3, real mode, reduce launches): the trailing
    // pure-copy rounds (an all-reduce's all-gather half) leave the rounds kernel
    // for the copy engines (bidirectional ring traffic 770 vs 660 GB/s/dir for SM
    // loads, profiles/r01/p2p_bidir.jsonl).  The kernel keeps rounds [0, k)
    // without a final barrier: the tail's first barrier (the peers of rounds k-1
    // and k, as inside the kernel) publishes them.  Tail tasks read and write the
    // reduction's result buffers only (no staging sets), so the kernels of later
    // buckets may run beside the tail.
    if (!pure && allow_tail && p->opts.copy_engine == 3 && ctx->mode == MODE_REAL) {
      int k = R;
      while (k > 0 && pure_round(k - 1)) --k;
      bool ok = k > 0 && k < R;
      auto result_buf = [](int kind) { return kind == BUF_GHAT || kind == BUF_GSHARD; };
      for (int r = k; r < R && ok; ++r)
        for (int x = 0; x < pl.N && ok; ++x)
          for (const Task& t : L.rounds[r][x]) ok = ok && result_buf(t.dst.kind) && result_buf(t.in[0].kind);
      if (ok) {
        DevLaunch tl;
        tl.dma = true;
        tl.copies.assign(R - k, {});
        tl.round_peers.assign(R - k, 0);
        for (int r = k; r < R; ++r) {
          for (const Task& t : L.rounds[r][ctx->rank]) {
            const DTask d = resolve(p, t, ctx->rank, -1, win_shift);
            tl.copies[r - k].push_back({d.dst, d.in[0], (size_t)t.n * pl.esz[t.dst.kind]});
          }
          tl.round_peers[r - k] = L.barrier_peers(r, ctx->rank);
          tl.bytes += bytes_r[r];
          tl.hbm += hbm_r[r];
        }
        tl.final_barrier = dl.final_barrier;
        tl.final_peers = dl.final_peers;
        dl.nrounds = k;
        dl.final_barrier = 0;
        dl.final_peers = 0;
        dl.bytes -= tl.bytes;
        dl.hbm -= tl.hbm;
        dl.tail.push_back(std::move(tl));
      }
    }
    if (pure) {
      dl.dma = true;
      dl.copies.assign(R, {});
      dl.round_peers.assign(R, 0);
      for (int r = 0; r < R; ++r) {
        for (int x = 0; x < pl.N; ++x) {
          if (ctx->mode == MODE_REAL && x != ctx->rank) continue;
          for (const Task& t : L.rounds[r][x]) {
            const DTask d = resolve(p, t, x, -1, win_shift);
            dl.copies[r].push_back({d.dst, d.in[0], (size_t)t.n * pl.esz[t.dst.kind]});
          }
        }
        dl.round_peers[r] = (ctx->mode == MODE_REAL) ? L.barrier_peers(r, ctx->rank) : 0;
      }
    }
    return dl;
  };
  // copies of raw gradient chunks (no round barriers: the data is immutable in a step)
  auto build_copies = [&](const Launch& L) {
    DevLaunch dl;
    dl.dma = true;
    dl.copies.assign(L.rounds.size(), {});
    dl.round_peers.assign(L.rounds.size(), 0);
    for (size_t r = 0; r < L.rounds.size(); ++r)
      for (int x = 0; x < pl.N; ++x) {
        if (ctx->mode == MODE_REAL && x != ctx->rank) continue;
        for (const Task& t : L.rounds[r][x]) {
          const DTask d = resolve(p, t, x, -1);
          dl.copies[r].push_back({d.dst, d.in[0], (size_t)t.n * 2});
          if (t.in[0].rank != x) dl.bytes += 2 * t.n;
          dl.hbm += 4 * t.n;
        }
      }
    return dl;
  };
  p->red_pre.clear();
  p->acc_pre.clear();
  p->red.clear();
  p->gat.clear();
  p->acc_first.clear();
  p->acc_next.clear();
  p->red_acc.clear();
  p->win.assign(pl.buf_len[BUF_WIN] > 0 ? pl.opt.windows : 0, {});
  for (const BucketSchedule& S : pl.sched) {
    p->red.push_back(build(S.reduce, -1, 0, true));
    p->gat.push_back(build(S.gather, -1));
    for (int w = 0; w < (int)p->win.size(); ++w) p->win[w].push_back(build(S.window, -1, int64_t(w) * pl.B));
    if (!S.reduce_pre.rounds.empty()) p->red_pre.push_back(build_copies(S.reduce_pre));
    if (!S.accum_pre.rounds.empty()) p->acc_pre.push_back(build_copies(S.accum_pre));
    if (pl.opt.accum) {
      p->acc_first.push_back(build(S.accum, -1));
      p->acc_next.push_back(build(S.accum, pl.acc_kind));
      p->red_acc.push_back(build(S.reduce_acc, -1));
    }
  }
  // bounds check of every resolved device span against the regions it must
  // lie in (compute-sanitizer is closed on this pool: our own check, on the
  // host, before any kernel can touch a bad address)
  {
    const size_t rb = kHeaderBytes + (size_t)pl.region_bytes;
    auto inside = [&](const void* ptr, size_t bytes) {
      const char* c = static_cast<const char*>(ptr);
      for (char* base : p->peer_base)
        if (base && c >= base + kHeaderBytes && c + bytes <= base + rb) return true;
      return false;
    };
    for (const DTask& d : tasks) {
      const size_t n = (size_t)d.n8 * 8;
      bool ok = inside(d.dst, n * (d.out_f32 ? 4 : 2));
      for (int i = 0; i < d.nin && ok; ++i) ok = inside(d.in[i], n * (((d.f32mask >> i) & 1u) ? 4 : 2));
      if (!ok) return fail(PARO_ERR_INVALID, "internal error: a collective task addresses memory outside the plan's regions");
    }
  }
  if (!rounds.empty()) {
    CK(cudaMalloc(&p->d_rounds, rounds.size() * sizeof(DRound)));
    CK(cudaMemcpy(p->d_rounds, rounds.data(), rounds.size() * sizeof(DRound), cudaMemcpyHostToDevice));
  }
  if (!tasks.empty()) {
    CK(cudaMalloc(&p->d_tasks, tasks.size() * sizeof(DTask)));
    CK(cudaMemcpy(p->d_tasks, tasks.data(), tasks.size() * sizeof(DTask), cudaMemcpyHostToDevice));
  }
  return PARO_OK;
}

// Record the start event of a timed launch; returns the slot or -1.
int prof_begin(PlanT* p, cudaStream_t s, int kind, int64_t amount, int64_t hbm = 0) {
  if (!p->prof || 2 * (p->prof_used + 1) > (int)p->prof_ev.size()) return -1;
  const int k = p->prof_used++;
  p->prof_kind[k] = kind;
  p->prof_amount[k] = amount;
  p->prof_hbm[k] = hbm;
  cudaEventRecord(p->prof_ev[2 * k], s);
  return k;
}
void prof_end(PlanT* p, cudaStream_t s, int k) {
  if (k >= 0) cudaEventRecord(p->prof_ev[2 * k + 1], s);
}

constexpr int kTraceLaunches = 512;

// CTAs of a collective launch: comm_ctas, or (0) one per SM.  Sizing small
// launches down (~4 tiles per CTA) was measured slower at every size (1 MiB
// all-reduce, 2 GPUs: one-shot 21.2 vs 19.2 us, HO 35.9 vs 31.9 us; 4 GPUs the
// same direction, profiles/r02/latency_*): more CTAs put more loads in flight
// and the entry barrier has no grid arrival
int comm_grid(const PlanT* p) {
  int g = p->opts.comm_ctas > 0 ? p->opts.comm_ctas : p->ctx->sm_count;
  if (p->ctx->mode == MODE_REAL) {
    if (g > p->ctx->sm_count) g = p->ctx->sm_count;   // co-residency of all CTAs (barriers)
  } else {
    g = p->ctx->sm_count * 2;
  }
  return g;
}

// First barrier of a launch published by CTA 0 without a grid arrival (kernels.cu
// entry_barrier); PARO_ENTRY_BARRIER=0 restores the all-CTA arrival (A/B runs).
bool entry_fast_on() {
  static const bool on = !(std::getenv("PARO_ENTRY_BARRIER") && std::atoi(std::getenv("PARO_ENTRY_BARRIER")) == 0);
  return on;
}


// 1-CTA peer barrier on the second channel (stream s), for copy-engine launches.
// channel 2 (hdr + 1024: copy-engine launches, the gradient producer) or 3
// (hdr + 2048: the parameter consumer); each channel's launches run on one stream
paro_status_t barrier2(PlanT* p, uint64_t peers, cudaStream_t s, int* nlaunch, int channel = 2) {
  paro_ctx* ctx = p->ctx;
  if (ctx->mode != MODE_REAL || !peers) return PARO_OK;
  char* hdr = p->region[0] + (channel == 3 ? 1024 : 0);
  RoundsArgs a{};
  a.nrounds = 0;
  a.final_barrier = 1;
  a.final_peers = peers;
  a.entry_fast = entry_fast_on() ? 1 : 0;
  a.bar.peer_slot = channel == 3 ? p->d_peer_slot3 : p->d_peer_slot2;
  a.bar.my_flags = reinterpret_cast<uint64_t*>(hdr + 1024);
  a.bar.arrive = reinterpret_cast<unsigned long long*>(hdr + 1536);
  a.bar.go = reinterpret_cast<unsigned long long*>(hdr + 1544);
  a.bar.err = reinterpret_cast<int*>(p->region[0] + 520);
  a.bar.gen = reinterpret_cast<unsigned long long*>(hdr + 1552);
  a.bar.exitc = reinterpret_cast<unsigned int*>(hdr + 1560);
  CK(launch_rounds(a, 1, 32, s));
  ++*nlaunch;
  return PARO_OK;
}

// A pure-copy launch on the copy engines: barrier with the round's peers, then
// one cudaMemcpyAsync per copy (peer memory is mapped: NVLink P2P DMA).
paro_status_t run_dma_launch(PlanT* p, const DevLaunch& dl, cudaStream_t s, int* nlaunch) {
  paro_ctx* ctx = p->ctx;
  for (size_t r = 0; r < dl.copies.size(); ++r) {
    paro_status_t st = barrier2(p, dl.round_peers[r], s, nlaunch);
    if (st != PARO_OK) return st;
    const int k = prof_begin(p, s, 1, r == 0 ? dl.bytes : 0, r == 0 ? dl.hbm : 0);
    for (const CopyOp& c : dl.copies[r]) {
      CK(cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyDeviceToDevice, s));
      if (ctx->mode == MODE_REAL) {   // copy-engine transfer over NVLink: counted at enqueue
        const int rs = data_rank(p, c.src), rd = data_rank(p, c.dst);
        const int other = rs != ctx->rank ? rs : rd;
        if (other >= 0 && other != ctx->rank)
          p->moved_host[other / p->pl->M != ctx->rank / p->pl->M ? 1 : 0] += (int64_t)c.bytes;
      }
    }
    prof_end(p, s, k);
  }
  if (dl.final_barrier) return barrier2(p, dl.final_peers, s, nlaunch);
  return PARO_OK;
}

paro_status_t run_launch_kernel(PlanT* p, const DevLaunch& dl, int* nlaunch);

// Launch one collective (reduce or gather of one bucket) on the comm stream.
// A copy-engine tail follows on the dma stream: with `tail_on_dma` the caller
// orders the consumers after the dma stream itself (*tail_on_dma = true), else
// the comm stream waits for the tail here.
paro_status_t run_launch(PlanT* p, const DevLaunch& dl, int* nlaunch, bool* tail_on_dma = nullptr) {
  paro_ctx* ctx = p->ctx;
  if (dl.dma) return run_dma_launch(p, dl, ctx->comm, nlaunch);
  paro_status_t s = run_launch_kernel(p, dl, nlaunch);
  if (s != PARO_OK || dl.tail.empty()) return s;
  CK(cudaEventRecord(p->ev_tail, ctx->comm));
  CK(cudaStreamWaitEvent(ctx->dma, p->ev_tail, 0));
  s = run_dma_launch(p, dl.tail[0], ctx->dma, nlaunch);
  if (s != PARO_OK) return s;
  if (tail_on_dma) {
    *tail_on_dma = true;
  } else {
    CK(cudaEventRecord(p->ev_tail, ctx->dma));
    CK(cudaStreamWaitEvent(ctx->comm, p->ev_tail, 0));
  }
  return PARO_OK;
}

// The rounds-kernel part of a launch, on the comm stream.
paro_status_t run_launch_kernel(PlanT* p, const DevLaunch& dl, int* nlaunch) {
  paro_ctx* ctx = p->ctx;
  if (dl.nrounds == 0 && (!dl.final_barrier || ctx->mode != MODE_REAL)) return PARO_OK;
  const int grid = comm_grid(p);
  RoundsArgs a{};
  a.tasks = p->d_tasks;
  a.alpha = p->alpha;
  // emulated intra/inter gap: this rank's inter-group transfers are paced to
  // inter_gbps, spread evenly over the CTAs (real mode, TMA rounds kernel)
  a.inter_bytes_per_ns = (ctx->mode == MODE_REAL && p->opts.inter_gbps > 0.f)
                             ? (double)p->opts.inter_gbps / (double)grid : 0.0;
  if (ctx->mode == MODE_REAL) {
    char* hdr = p->region[0];
    a.rounds = p->d_rounds + dl.round_off;
    a.nrounds = dl.nrounds;
    a.final_barrier = dl.final_barrier;
    a.final_peers = dl.final_peers;
    a.entry_fast = entry_fast_on() ? 1 : 0;
    a.moved = p->d_moved;
    a.bar.peer_slot = p->d_peer_slot;
    a.bar.my_flags = reinterpret_cast<uint64_t*>(hdr);
    a.bar.arrive = reinterpret_cast<unsigned long long*>(hdr + 512);
    a.bar.go = reinterpret_cast<unsigned long long*>(hdr + 528);
    a.bar.err = reinterpret_cast<int*>(hdr + 520);
    a.bar.gen = reinterpret_cast<unsigned long long*>(hdr + 536);
    a.bar.exitc = reinterpret_cast<unsigned int*>(hdr + 544);
    a.sys_fence_all = p->pl->opt.push ? 1 : 0;
    const int k = prof_begin(p, ctx->comm, 1, dl.bytes, dl.hbm);
    if (p->prof && p->d_trace && (int)p->trace_nrounds.size() < kTraceLaunches) {
      a.trace = p->d_trace + (size_t)p->trace_nrounds.size() * ctx->sm_count * kTraceSlots;
      p->trace_nrounds.push_back(dl.nrounds);
      p->trace_grids.push_back(grid);
    }
    if (p->opts.comm_impl != 1) CK(launch_rounds_tma(a, grid, dl.max_in, ctx->comm, p->opts.comm_impl == 2, dl.generic));
    else CK(launch_rounds(a, grid, 0, ctx->comm));
    prof_end(p, ctx->comm, k);
    ++*nlaunch;
  } else {
    for (int r = 0; r < dl.nrounds; ++r) {
      a.rounds = p->d_rounds + dl.round_off + r;
      a.nrounds = 1;
      const int k = prof_begin(p, ctx->comm, 1, r == 0 ? dl.bytes : 0, r == 0 ? dl.hbm : 0);
      if (p->opts.comm_impl != 1) CK(launch_rounds_tma(a, grid, dl.max_in, ctx->comm, p->opts.comm_impl == 2, dl.generic));
      else CK(launch_rounds(a, grid, 0, ctx->comm));
      prof_end(p, ctx->comm, k);
      ++*nlaunch;
    }
  }
  return PARO_OK;
}

// Per-parameter caller gradients -> each local rank's flat gradient buffer
// (compute stream; the comm stream waits for it).
paro_status_t pack_grads(PlanT* p, const void* const* grads, int* launches) {
  paro_ctx* ctx = p->ctx;
  const Planner& pl = *p->pl;
  const int nl = (int)p->local.size();
  const int np = (int)pl.param_sizes.size();
  CK(cudaEventSynchronize(p->ev_pack_staged));   // staging buffer free again
  int k = 0;
  int64_t maxn = 0;
  for (int li = 0; li < nl; ++li) {
    const int r = p->local[li];
    for (int i = 0; i < np; ++i) {
      if (pl.param_sizes[i] == 0) continue;
      p->h_pack[k].src = static_cast<const uint16_t*>(grads[li * np + i]);
      p->h_pack[k].dst = reinterpret_cast<uint16_t*>(data_ptr(p, r, BUF_GRAD, pl.param_offsets[i]));
      p->h_pack[k].n = pl.param_sizes[i];
      maxn = std::max(maxn, pl.param_sizes[i]);
      ++k;
    }
  }
  CK(cudaMemcpyAsync(p->d_pack, p->h_pack, sizeof(PackEntry) * k, cudaMemcpyHostToDevice, ctx->comp));
  CK(cudaEventRecord(p->ev_pack_staged, ctx->comp));
  CK(launch_pack(p->d_pack, k, maxn, ctx->comp));
  ++*launches;
  CK(cudaEventRecord(p->ev_comp, ctx->comp));
  CK(cudaStreamWaitEvent(ctx->comm, p->ev_comp, 0));
  return PARO_OK;
}

// Step-end barrier with every peer (real mode, N > 1): after it no peer reads
// (fused Adam, pull rounds) or writes (push rounds) this rank's buffers any
// more, so the caller may overwrite its gradients and read its parameters.
paro_status_t all_peer_barrier(PlanT* p, int* launches) {
  paro_ctx* ctx = p->ctx;
  if (ctx->mode != MODE_REAL || p->pl->N <= 1 || p->pl->opt.topology == PARO_TOPO_NCCL) return PARO_OK;
  DevLaunch fin;
  fin.nrounds = 0;
  fin.final_barrier = 1;
  for (int x = 0; x < p->pl->N; ++x)
    if (x != ctx->rank) fin.final_peers |= uint64_t(1) << x;
  return run_launch(p, fin, launches);
}

ncclComm_t pick_comm(paro_ctx* ctx, NcclCall::Comm c) {
  return c == NcclCall::INTRA ? ctx->intra : (c == NcclCall::INTER ? ctx->inter : ctx->world);
}

paro_status_t run_nccl(PlanT* p, const std::vector<NcclCall>& calls) {
  paro_ctx* ctx = p->ctx;
  for (const NcclCall& c : calls) {
    void* send = data_ptr(p, c.send.rank, c.send.kind, c.send.off);
    void* recv = data_ptr(p, c.recv.rank, c.recv.kind, c.recv.off);
    ncclComm_t cm = pick_comm(ctx, c.comm);
    // bf16 wire: NCCL averages the raw gradients (ncclAvg); fp32 wire: the
    // bucket was pre-scaled into fp32 by the rounds kernel, NCCL sums; without
    // pre-division NCCL sums the raw gradients and Adam takes the average
    const bool f32 = p->pl->esz[c.send.kind] == 4;
    const ncclDataType_t dt = f32 ? ncclFloat : ncclBfloat16;
    const ncclRedOp_t op = (!f32 && p->pl->opt.predivide) ? ncclAvg : ncclSum;
    if (c.kind == NcclCall::RS) NK(ncclReduceScatter(send, recv, c.count, dt, op, cm, ctx->comm));
    else if (c.kind == NcclCall::AG) NK(ncclAllGather(send, recv, c.count, dt, cm, ctx->comm));
    else NK(ncclAllReduce(send, recv, c.count, dt, op, cm, ctx->comm));
  }
  return PARO_OK;
}

void destroy_plan(PlanT* p) {
  if (!p) return;
  paro_ctx* ctx = p->ctx;
  if (ctx && ctx->mode != MODE_PLANNER) {
    cudaSetDevice(ctx->device);
    if (p->stepped && p->last_stream) cudaStreamSynchronize(p->last_stream);
    if (ctx->mode == MODE_REAL) {
      for (int x = 0; x < (int)p->peer_base.size(); ++x)
        if (x != ctx->rank && p->peer_base[x]) cudaIpcCloseMemHandle(p->peer_base[x]);
    }
    for (char* r : p->region) cudaFree(r);
    cudaFree(p->d_peer_slot);
    cudaFree(p->d_peer_slot2);
    cudaFree(p->d_peer_slot3);
    if (p->ev_cons) cudaEventDestroy(p->ev_cons);
    for (cudaEvent_t e : p->ev_pfinal) if (e) cudaEventDestroy(e);
    cudaFree(p->d_rounds);
    cudaFree(p->d_tasks);
    cudaFree(p->d_partials);
    cudaFree(p->d_norm);
    cudaFree(p->d_nonfinite);
    cudaFree(p->d_sg);
    cudaFree(p->d_skip);
    cudaFree(p->d_moved);
    cudaFree(p->d_pack);
    if (p->h_pack) cudaFreeHost(p->h_pack);
    for (cudaEvent_t e : {p->ev_fork, p->ev_comm, p->ev_comp, p->ev_pack_staged, p->ev_unpack_staged, p->ev_dma,
                          p->ev_tail})
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : p->prof_ev) cudaEventDestroy(e);
    cudaFree(p->d_trace);
    for (cudaEvent_t e : p->ev_red) cudaEventDestroy(e);
    for (cudaEvent_t e : p->ev_pre) cudaEventDestroy(e);
    for (cudaEvent_t e : p->ev_prod) if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : p->ev_adam) cudaEventDestroy(e);
  }
  delete p;
}

paro_status_t make_streams(paro_ctx* ctx) {
  CK(cudaSetDevice(ctx->device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, ctx->device));
  ctx->sm_count = prop.multiProcessorCount;
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CK(cudaStreamCreateWithFlags(&ctx->main, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithPriority(&ctx->comm, cudaStreamNonBlocking, hi));  // collectives first
  CK(cudaStreamCreateWithFlags(&ctx->comp, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithPriority(&ctx->dma, cudaStreamNonBlocking, hi));
  CK(cudaStreamCreateWithFlags(&ctx->sink, cudaStreamNonBlocking));
  return PARO_OK;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

const char* paro_last_error(void) { return g_last_error.c_str(); }

const char* paro_version(void) { return "paro-b200 0.1.0 sm_100a"; }

void paro_opts_default(paro_opts_t* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->bucket_elems = int64_t(1) << 26;
  o->topology = PARO_TOPO_HO_RING;
  o->beta1 = 0.9f;
  o->beta2 = 0.95f;
  o->eps = 1e-8f;
  o->weight_decay = 0.0f;
  o->loss_scale = 1.0f;
  o->comm_ctas = 0;
  o->pipeline_depth = 2;
  o->pull_transport = 1;
  o->adam_impl = 0;
  o->comm_impl = 2;
  o->inter_gbps = 0.f;
  o->grad_accum = 0;
  o->clip_norm = 0.f;
  o->skip_nonfinite = 0;
  o->gather_windows = 0;
  o->fuse_gather = 1;
  o->copy_engine = 0;
  o->stream = nullptr;
  o->frozen = 0;
  o->grad_slots = 0;
  o->fuse_allreduce = 1;
  o->adam_smem_kb = 0;
  o->wire_dtype = 0;
  o->predivide = 1;
  o->bucket_groups = nullptr;
  o->n_bucket_groups = 0;
}

paro_status_t paro_get_unique_id(paro_uid_t* out) {
  if (!out) return fail(PARO_ERR_INVALID, "null uid");
  static_assert(sizeof(ncclUniqueId) <= sizeof(paro_uid_t), "uid size");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(PARO_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  std::memset(out, 0, sizeof(*out));
  std::memcpy(out->bytes, &id, sizeof(id));
  return PARO_OK;
}

paro_status_t paro_init_planner(int world_size, int group_size, paro_ctx_t* out) {
  if (!out) return fail(PARO_ERR_INVALID, "null out");
  std::string e = validate_cluster(world_size, group_size);
  if (!e.empty()) return fail(PARO_ERR_INVALID, e);
  auto* c = new paro_ctx();
  c->mode = MODE_PLANNER;
  c->N = world_size;
  c->M = group_size;
  *out = c;
  return PARO_OK;
}

paro_status_t paro_init_emulated(int world_size, int group_size, int device, paro_ctx_t* out) {
  if (!out) return fail(PARO_ERR_INVALID, "null out");
  std::string e = validate_cluster(world_size, group_size);
  if (!e.empty()) return fail(PARO_ERR_INVALID, e);
  if (world_size > kMaxAdamSegs) return fail(PARO_ERR_INVALID, "emulated mode supports world_size <= 16");
  auto* c = new paro_ctx();
  c->mode = MODE_EMU;
  c->N = world_size;
  c->M = group_size;
  c->device = device;
  paro_status_t st = make_streams(c);
  if (st != PARO_OK) {
    delete c;
    return st;
  }
  *out = c;
  return PARO_OK;
}

paro_status_t paro_init(int world_size, int group_size, int rank, const paro_uid_t* uid, int device,
                        paro_ctx_t* out) {
  if (!out || !uid) return fail(PARO_ERR_INVALID, "null argument");
  std::string e = validate_cluster(world_size, group_size);
  if (!e.empty()) return fail(PARO_ERR_INVALID, e);
  if (rank < 0 || rank >= world_size) return fail(PARO_ERR_INVALID, "rank out of range");
  auto* c = new paro_ctx();
  c->mode = MODE_REAL;
  c->N = world_size;
  c->M = group_size;
  c->rank = rank;
  c->device = device;
  paro_status_t st = make_streams(c);
  if (st != PARO_OK) {
    delete c;
    return st;
  }
  if (world_size > 1) {
    ncclUniqueId id;
    std::memcpy(&id, uid->bytes, sizeof(id));
    paro_ctx* ctx = c;
    ncclResult_t r = ncclCommInitRank(&c->world, world_size, id, rank);
    if (r != ncclSuccess) {
      delete c;
      return fail(PARO_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    const int j = rank / group_size, p = rank % group_size;
    NK(ncclCommSplit(c->world, j, p, &c->intra, nullptr));
    NK(ncclCommSplit(c->world, p, j, &c->inter, nullptr));
  }
  *out = c;
  return PARO_OK;
}

paro_status_t paro_finalize(paro_ctx_t ctx) {
  if (!ctx) return PARO_OK;
  if (ctx->mode != MODE_PLANNER) {
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();
    if (ctx->intra) ncclCommDestroy(ctx->intra);
    if (ctx->inter) ncclCommDestroy(ctx->inter);
    if (ctx->world) ncclCommDestroy(ctx->world);
    for (cudaStream_t s : {ctx->main, ctx->comm, ctx->comp, ctx->dma, ctx->sink})
      if (s) cudaStreamDestroy(s);
  }
  delete ctx;
  return PARO_OK;
}

paro_status_t paro_plan(paro_ctx_t ctx, const char* strategy, const int64_t* param_sizes, int n_params,
                        const paro_opts_t* opts, paro_plan_t* out) {
  paro_status_t st = check_ctx(ctx);
  if (st != PARO_OK) return st;
  if (!strategy || !out || (n_params > 0 && !param_sizes) || n_params < 0)
    return fail(PARO_ERR_INVALID, "null argument");
  paro_opts_t o;
  if (opts) o = *opts;
  else paro_opts_default(&o);
  if (o.topology == PARO_TOPO_NCCL && ctx->mode == MODE_EMU)
    return fail(PARO_ERR_INVALID, "NCCL topology needs real ranks");
  if (o.comm_ctas < 0) o.comm_ctas = 0;
  std::vector<int64_t> sizes(param_sizes, param_sizes + n_params);
  PlanOptions po;
  po.bucket_elems = o.bucket_elems > 0 ? o.bucket_elems : (int64_t(1) << 26);
  po.topology = o.topology;
  po.pipeline_depth = o.pipeline_depth > 0 ? o.pipeline_depth : 2;
  po.push = o.pull_transport == 0;
  po.fuse_final = !(o.inter_gbps > 0.f);   // paced runs keep every transfer in the rounds kernel
  po.accum = o.grad_accum != 0;
  if (o.clip_norm < 0.f) return fail(PARO_ERR_INVALID, "clip_norm must be >= 0");
  po.two_phase = o.clip_norm > 0.f || o.skip_nonfinite != 0;
  if (po.two_phase) po.fuse_final = false;   // g_hat is materialised for the norm pass
  po.fuse_ar_e = po.fuse_final && o.fuse_allreduce != 0;
  if (o.fuse_allreduce == 0) po.fuse_final = false;   // no part of the reduction inside Adam
  if (o.gather_windows < 0 || o.gather_windows > 64) return fail(PARO_ERR_INVALID, "gather_windows must be in [0, 64]");
  po.windows = o.gather_windows;
  if (o.fuse_gather < 0 || o.fuse_gather > 2) return fail(PARO_ERR_INVALID, "fuse_gather must be 0, 1 or 2");
  if (o.comm_impl < 0 || o.comm_impl > 2) return fail(PARO_ERR_INVALID, "comm_impl must be 0, 1 or 2");
  if (o.adam_impl < 0 || o.adam_impl > 4) return fail(PARO_ERR_INVALID, "adam_impl must be 0 .. 4");
  if (o.adam_smem_kb < 0 || o.adam_smem_kb > 220) return fail(PARO_ERR_INVALID, "adam_smem_kb must be in [0, 220]");
  po.fuse_gather = (o.inter_gbps > 0.f || o.topology == PARO_TOPO_NCCL) ? 0 : o.fuse_gather;
  // paced (emulated-gap) runs keep every transfer in the rounds kernel, which
  // paces them; the NCCL comparator has no copy-engine path
  if (o.inter_gbps > 0.f || o.topology == PARO_TOPO_NCCL) o.copy_engine = 0;
  if (o.copy_engine < 0 || o.copy_engine > 3) return fail(PARO_ERR_INVALID, "copy_engine must be 0 .. 3");
  po.ce_reduce = o.copy_engine == 2;
  po.params_only = o.frozen != 0;
  if (o.grad_slots < 0) return fail(PARO_ERR_INVALID, "grad_slots must be >= 0");
  if (o.grad_slots > 0 && o.grad_accum) return fail(PARO_ERR_INVALID, "grad_slots cannot be combined with grad_accum");
  if (o.grad_slots > 0) o.copy_engine = 0;   // its stream and barrier channel produce the gradients
  po.grad_slots = o.frozen ? 0 : o.grad_slots;
  po.ce_reduce = o.copy_engine == 2;
  if (o.wire_dtype != 0 && o.wire_dtype != 1) return fail(PARO_ERR_INVALID, "wire_dtype must be 0 (bf16) or 1 (fp32)");
  po.wire = o.wire_dtype == 1 ? 4 : 2;
  po.predivide = o.predivide != 0;
  if (o.n_bucket_groups < 0 || (o.n_bucket_groups > 0 && !o.bucket_groups))
    return fail(PARO_ERR_INVALID, "bucket_groups: null pointer or negative count");
  for (int k = 0; k < o.n_bucket_groups; ++k) po.groups.push_back(o.bucket_groups[k]);
  o.bucket_groups = nullptr;   // not kept: the planner holds its copy
  o.n_bucket_groups = 0;
  auto* p = new PlanT();
  p->ctx = ctx;
  p->opts = o;
  p->alpha = po.predivide ? (float)(1.0 / (double)ctx->N) : 1.0f;
  try {
    p->pl.reset(new Planner(ctx->N, ctx->M, strategy, sizes, po));
  } catch (const std::exception& ex) {
    delete p;
    return fail(PARO_ERR_INVALID, ex.what());
  }
  if (ctx->mode == MODE_PLANNER) {
    *out = p;
    return PARO_OK;
  }
  const Planner& pl = *p->pl;
  const int N = pl.N;
  const size_t region_bytes = kHeaderBytes + (size_t)pl.region_bytes;
  auto bail = [&](paro_status_t s) {
    destroy_plan(p);
    return s;
  };
#define PCK(call)                                                  \
  do {                                                             \
    cudaError_t e_ = (call);                                       \
    if (e_ != cudaSuccess) return bail(cuda_fail(ctx, #call, e_)); \
  } while (0)
  if (ctx->mode == MODE_REAL) p->local = {ctx->rank};
  else
    for (int r = 0; r < N; ++r) p->local.push_back(r);
  p->peer_base.assign(N, nullptr);
  for (int r : p->local) {
    char* base = nullptr;
    PCK(cudaMalloc(&base, region_bytes));
    PCK(cudaMemset(base, 0, region_bytes));
    p->region.push_back(base);
    p->peer_base[r] = base;
  }
  if (ctx->mode == MODE_REAL && N > 1) {
    // exchange IPC handles of the symmetric regions over the world communicator
    cudaIpcMemHandle_t h;
    PCK(cudaIpcGetMemHandle(&h, p->region[0]));
    char* d_h = nullptr;
    PCK(cudaMalloc(&d_h, sizeof(h) * (N + 1)));
    PCK(cudaMemcpy(d_h + sizeof(h) * N, &h, sizeof(h), cudaMemcpyHostToDevice));
    ncclResult_t r = ncclAllGather(d_h + sizeof(h) * N, d_h, sizeof(h), ncclChar, ctx->world, ctx->main);
    if (r != ncclSuccess) {
      cudaFree(d_h);
      return bail(nccl_fail(ctx, "ncclAllGather(ipc handles)", r));
    }
    PCK(cudaStreamSynchronize(ctx->main));
    std::vector<cudaIpcMemHandle_t> hs(N);
    PCK(cudaMemcpy(hs.data(), d_h, sizeof(h) * N, cudaMemcpyDeviceToHost));
    cudaFree(d_h);
    for (int x = 0; x < N; ++x) {
      if (x == ctx->rank) continue;
      void* ptr = nullptr;
      PCK(cudaIpcOpenMemHandle(&ptr, hs[x], cudaIpcMemLazyEnablePeerAccess));
      p->peer_base[x] = static_cast<char*>(ptr);
    }
    std::vector<uint64_t*> slots(64, nullptr);
    for (int x = 0; x < N; ++x) slots[x] = reinterpret_cast<uint64_t*>(p->peer_base[x]) + ctx->rank;
    PCK(cudaMalloc(&p->d_peer_slot, 64 * sizeof(uint64_t*)));
    PCK(cudaMemcpy(p->d_peer_slot, slots.data(), 64 * sizeof(uint64_t*), cudaMemcpyHostToDevice));
    for (int x = 0; x < N; ++x) slots[x] = reinterpret_cast<uint64_t*>(p->peer_base[x] + 1024) + ctx->rank;
    PCK(cudaMalloc(&p->d_peer_slot2, 64 * sizeof(uint64_t*)));
    PCK(cudaMemcpy(p->d_peer_slot2, slots.data(), 64 * sizeof(uint64_t*), cudaMemcpyHostToDevice));
    for (int x = 0; x < N; ++x) slots[x] = reinterpret_cast<uint64_t*>(p->peer_base[x] + 2048) + ctx->rank;
    PCK(cudaMalloc(&p->d_peer_slot3, 64 * sizeof(uint64_t*)));
    PCK(cudaMemcpy(p->d_peer_slot3, slots.data(), 64 * sizeof(uint64_t*), cudaMemcpyHostToDevice));
  }
  {
    paro_status_t s2 = upload_schedule(p);
    if (s2 != PARO_OK) return bail(s2);
  }
  const int nb = (int)pl.buckets.size();
  p->partials_cap = adam_grid() * ((pl.N == 1 && pl.opt.grad_slots == 0) ? 1 : nb);
  PCK(cudaMalloc(&p->d_partials, sizeof(double) * p->partials_cap));
  PCK(cudaMalloc(&p->d_norm, sizeof(double)));
  PCK(cudaMemset(p->d_norm, 0, sizeof(double)));
  PCK(cudaMalloc(&p->d_nonfinite, sizeof(int)));
  PCK(cudaMemset(p->d_nonfinite, 0, sizeof(int)));
  PCK(cudaMalloc(&p->d_sg, sizeof(float)));
  PCK(cudaMalloc(&p->d_skip, sizeof(int)));
  PCK(cudaMemset(p->d_skip, 0, sizeof(int)));
  PCK(cudaMalloc(&p->d_moved, 2 * sizeof(unsigned long long)));
  PCK(cudaMemset(p->d_moved, 0, 2 * sizeof(unsigned long long)));
  p->pack_cap = std::max(1, n_params) * (int)p->local.size();
  PCK(cudaMalloc(&p->d_pack, 2 * sizeof(PackEntry) * p->pack_cap));   // [pack | unpack]
  PCK(cudaHostAlloc(&p->h_pack, 2 * sizeof(PackEntry) * p->pack_cap, cudaHostAllocDefault));
  for (cudaEvent_t* e : {&p->ev_fork, &p->ev_comm, &p->ev_comp, &p->ev_pack_staged, &p->ev_unpack_staged,
                        &p->ev_dma, &p->ev_tail})
    PCK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  p->ev_red.resize(nb);
  p->ev_adam.resize(nb);
  p->ev_pre.resize(nb);
  p->ev_prod.resize(nb);
  p->ev_pfinal.resize(nb);
  PCK(cudaEventCreateWithFlags(&p->ev_cons, cudaEventDisableTiming));
  for (int b = 0; b < nb; ++b) {
    PCK(cudaEventCreateWithFlags(&p->ev_red[b], cudaEventDisableTiming));
    PCK(cudaEventCreateWithFlags(&p->ev_pre[b], cudaEventDisableTiming));
    PCK(cudaEventCreateWithFlags(&p->ev_prod[b], cudaEventDisableTiming));
    PCK(cudaEventCreateWithFlags(&p->ev_pfinal[b], cudaEventDisableTiming));
    PCK(cudaEventCreateWithFlags(&p->ev_adam[b], cudaEventDisableTiming));
  }
  PCK(cudaDeviceSynchronize());
#undef PCK
  *out = p;
  return PARO_OK;
}

paro_status_t paro_plan_masked(paro_ctx_t ctx, const char* strategy, const int64_t* param_sizes,
                               const uint8_t* trainable, int n_params, const paro_opts_t* opts,
                               paro_plan_t* out_trainable, paro_plan_t* out_frozen) {
  if (!out_trainable || !out_frozen || !trainable || (n_params > 0 && !param_sizes) || n_params < 0)
    return fail(PARO_ERR_INVALID, "null argument");
  *out_trainable = nullptr;
  *out_frozen = nullptr;
  std::vector<int64_t> tr, fr;
  for (int i = 0; i < n_params; ++i) (trainable[i] ? tr : fr).push_back(param_sizes[i]);
  if (tr.empty()) return fail(PARO_ERR_INVALID, "no trainable tensor");
  paro_opts_t o;
  if (opts) o = *opts;
  else paro_opts_default(&o);
  o.frozen = 0;
  // layer-aligned buckets: a group boundary at tensor t becomes, in each
  // sub-list, the number of that list's tensors before t (empty groups merge)
  std::vector<int64_t> gt, gf;
  if (o.n_bucket_groups > 0 && o.bucket_groups) {
    for (int k = 0; k < o.n_bucket_groups; ++k) {
      const int64_t t = o.bucket_groups[k];
      if (t < 0 || t > n_params) return fail(PARO_ERR_INVALID, "bucket_groups: tensor index out of range");
      int64_t a = 0, b = 0;
      for (int64_t i = 0; i < t; ++i) (trainable[i] ? a : b) += 1;
      if (a < (int64_t)tr.size() && (gt.empty() || gt.back() < a)) gt.push_back(a);
      if (b < (int64_t)fr.size() && (gf.empty() || gf.back() < b)) gf.push_back(b);
    }
    if (gt.empty() || gt[0] != 0) gt.insert(gt.begin(), 0);
    if (!fr.empty() && (gf.empty() || gf[0] != 0)) gf.insert(gf.begin(), 0);
    o.bucket_groups = gt.data();
    o.n_bucket_groups = (int)gt.size();
  }
  paro_status_t st = paro_plan(ctx, strategy, tr.data(), (int)tr.size(), &o, out_trainable);
  if (st != PARO_OK || fr.empty()) return st;
  o.frozen = 1;
  if (o.n_bucket_groups > 0) {
    o.bucket_groups = gf.data();
    o.n_bucket_groups = (int)gf.size();
  }
  st = paro_plan(ctx, strategy, fr.data(), (int)fr.size(), &o, out_frozen);
  if (st != PARO_OK) {
    const std::string msg = g_last_error;
    paro_plan_destroy(*out_trainable);
    *out_trainable = nullptr;
    g_last_error = msg;
  }
  return st;
}

paro_status_t paro_plan_info(paro_plan_t p, paro_plan_info_t* out) {
  if (!p || !out) return fail(PARO_ERR_INVALID, "null argument");
  const Planner& pl = *p->pl;
  std::memset(out, 0, sizeof(*out));
  out->psi = pl.psi;
  out->psi_pad = pl.psi_pad;
  out->bucket_elems = pl.B;
  out->n_buckets = (int64_t)pl.buckets.size();
  out->p_numel = pl.p_numel;
  out->g_numel = pl.g_numel;
  out->os_numel = pl.os_numel;
  out->mem_p_bytes = pl.mem_bytes(0);
  out->mem_g_bytes = pl.mem_bytes(1);
  out->mem_os_bytes = pl.mem_bytes(2);
  int64_t ws = 0;
  for (int k = BUF_GHAT; k < BUF_NKINDS; ++k) ws += (int64_t)pl.esz[k] * pl.buf_len[k];
  out->workspace_bytes = ws + kHeaderBytes;
  out->grad_buffer_bytes = 2 * pl.buf_len[BUF_GRAD];
  const int me = p->ctx->mode == MODE_REAL ? p->ctx->rank : 0;
  out->step_send_bytes_intra = pl.send_intra[me];
  out->step_send_bytes_inter = pl.send_inter[me];
  out->n_rounds = pl.n_rounds;
  out->n_comm_launches = pl.n_comm_launches;
  if (pl.opt.accum) {
    out->accum_send_bytes_intra = pl.acc_send_intra[me];
    out->accum_send_bytes_inter = pl.acc_send_inter[me];
    out->accum_step_send_bytes_intra = pl.accstep_send_intra[me];
    out->accum_step_send_bytes_inter = pl.accstep_send_inter[me];
  }
  return PARO_OK;
}

paro_status_t paro_shard_range(paro_plan_t p, int state, int rank, int64_t bucket, int64_t* begin,
                               int64_t* end) {
  if (!p || !begin || !end) return fail(PARO_ERR_INVALID, "null argument");
  const Planner& pl = *p->pl;
  if (state < 0 || state > 2) return fail(PARO_ERR_INVALID, "state must be 0 (P), 1 (G) or 2 (OS)");
  if (rank < 0 || rank >= pl.N) return fail(PARO_ERR_INVALID, "rank out of range");
  if (bucket < 0 || bucket >= (int64_t)pl.buckets.size()) return fail(PARO_ERR_INVALID, "bucket out of range");
  const Level l = state == 0 ? pl.P : (state == 1 ? pl.G : pl.OS);
  pl.residency(l, rank, bucket, begin, end);
  return PARO_OK;
}

paro_status_t paro_bucket_range(paro_plan_t p, int64_t bucket, int64_t* begin, int64_t* end) {
  if (!p || !begin || !end) return fail(PARO_ERR_INVALID, "null argument");
  const Planner& pl = *p->pl;
  if (bucket < 0 || bucket >= (int64_t)pl.buckets.size()) return fail(PARO_ERR_INVALID, "bucket out of range");
  *begin = pl.buckets[bucket].first;
  *end = *begin + pl.buckets[bucket].second;
  return PARO_OK;
}

paro_status_t paro_rank_send_bytes(paro_plan_t p, int rank, int64_t* intra, int64_t* inter) {
  if (!p || !intra || !inter) return fail(PARO_ERR_INVALID, "null argument");
  if (rank < 0 || rank >= p->pl->N) return fail(PARO_ERR_INVALID, "rank out of range");
  *intra = p->pl->send_intra[rank];
  *inter = p->pl->send_inter[rank];
  return PARO_OK;
}

paro_status_t paro_rank_accum_send_bytes(paro_plan_t p, int rank, int64_t* acc_intra, int64_t* acc_inter,
                                         int64_t* step_intra, int64_t* step_inter) {
  if (!p || !acc_intra || !acc_inter || !step_intra || !step_inter) return fail(PARO_ERR_INVALID, "null argument");
  if (rank < 0 || rank >= p->pl->N) return fail(PARO_ERR_INVALID, "rank out of range");
  if (!p->pl->opt.accum) return fail(PARO_ERR_STATE, "plan was created without grad_accum");
  *acc_intra = p->pl->acc_send_intra[rank];
  *acc_inter = p->pl->acc_send_inter[rank];
  *step_intra = p->pl->accstep_send_intra[rank];
  *step_inter = p->pl->accstep_send_inter[rank];
  return PARO_OK;
}

paro_status_t paro_rank_gather_send_bytes(paro_plan_t p, int rank, int64_t* intra, int64_t* inter) {
  if (!p || !intra || !inter) return fail(PARO_ERR_INVALID, "null argument");
  if (rank < 0 || rank >= p->pl->N) return fail(PARO_ERR_INVALID, "rank out of range");
  *intra = p->pl->win_send_intra[rank];
  *inter = p->pl->win_send_inter[rank];
  return PARO_OK;
}

paro_status_t paro_bucket_gather_send_bytes(paro_plan_t p, int rank, int64_t bucket, int64_t* intra, int64_t* inter) {
  if (!p || !intra || !inter) return fail(PARO_ERR_INVALID, "null argument");
  if (rank < 0 || rank >= p->pl->N) return fail(PARO_ERR_INVALID, "rank out of range");
  if (bucket < 0 || bucket >= (int64_t)p->pl->buckets.size()) return fail(PARO_ERR_INVALID, "bucket out of range");
  *intra = p->pl->win_bucket_intra[bucket][rank];
  *inter = p->pl->win_bucket_inter[bucket][rank];
  return PARO_OK;
}

paro_status_t paro_buffer(paro_plan_t p, int rank, int kind, void** ptr) {
  if (!p || !ptr) return fail(PARO_ERR_INVALID, "null argument");
  paro_ctx* ctx = p->ctx;
  if (ctx->mode == MODE_PLANNER) return fail(PARO_ERR_STATE, "planning-only context has no buffers");
  if (!is_local(p, rank)) return fail(PARO_ERR_INVALID, "rank is not local to this process");
  const Planner& pl = *p->pl;
  if (kind == 0) *ptr = pl.opt.params_only ? nullptr : data_ptr(p, rank, BUF_GRAD, 0);
  else if (kind == 1) *ptr = data_ptr(p, rank, BUF_PARAM, 0);
  else if (kind == 2) *ptr = (pl.G == LV_N) ? nullptr : data_ptr(p, rank, BUF_GSHARD, 0);
  else if (kind == 3) *ptr = pl.buf_len[BUF_GHAT] ? data_ptr(p, rank, BUF_GHAT, 0) : nullptr;
  else if (kind == 4) *ptr = pl.buf_len[BUF_GACC] ? data_ptr(p, rank, BUF_GACC, 0) : nullptr;
  else if (kind == 5) *ptr = pl.buf_len[BUF_WIN] ? data_ptr(p, rank, BUF_WIN, 0) : nullptr;
  else return fail(PARO_ERR_INVALID, "kind must be 0 .. 5");
  return PARO_OK;
}

static paro_status_t opt_init_impl(paro_plan_t p, int rank, const float* src, uint64_t key,
                                   const paro_opt_state_t* st) {
  paro_ctx* ctx = p->ctx;
  paro_status_t s = check_ctx(ctx);
  if (s != PARO_OK) return s;
  if (ctx->mode == MODE_PLANNER) return fail(PARO_ERR_STATE, "planning-only context");
  const Planner& pl = *p->pl;
  if (!pl.opt.params_only && pl.os_numel > 0 && (!st || !st->master || !st->m || !st->v))
    return fail(PARO_ERR_INVALID, "null opt state");
  if (!is_local(p, rank)) return fail(PARO_ERR_INVALID, "rank is not local to this process");
  uint16_t* pbuf = reinterpret_cast<uint16_t*>(data_ptr(p, rank, BUF_PARAM, 0));
  for (size_t b = 0; b < pl.buckets.size(); ++b) {
    int64_t ob, oe, pb, pe;
    pl.residency(pl.OS, rank, b, &ob, &oe);
    pl.residency(pl.P, rank, b, &pb, &pe);
    const int64_t os_off = pl.buckets[b].first / pl.divl(pl.OS);
    const int64_t p_off = pl.buckets[b].first / pl.divl(pl.P);
    if (!pl.opt.params_only)
      CK(launch_init_range(src, key, ob, oe - ob, pl.bucket_real_end[b], st->master + os_off, st->m + os_off, st->v + os_off,
                           nullptr, ctx->main));
    CK(launch_init_range(src, key, pb, pe - pb, pl.bucket_real_end[b], nullptr, nullptr, nullptr, pbuf + p_off,
                         ctx->main));
  }
  CK(cudaStreamSynchronize(ctx->main));
  return PARO_OK;
}

paro_status_t paro_opt_state_init(paro_plan_t p, int rank, const float* master_full, const paro_opt_state_t* st) {
  if (!p) return fail(PARO_ERR_INVALID, "null plan");
  if (!master_full) return fail(PARO_ERR_INVALID, "null master vector");
  return opt_init_impl(p, rank, master_full, 0, st);
}

paro_status_t paro_opt_state_init_synth(paro_plan_t p, int rank, uint64_t seed, const paro_opt_state_t* st) {
  if (!p) return fail(PARO_ERR_INVALID, "null plan");
  return opt_init_impl(p, rank, nullptr, synth_key(seed, kTagMaster, 0, 0), st);
}

paro_status_t paro_synth_grads(paro_plan_t p, int rank, uint64_t seed, int64_t step) {
  if (!p) return fail(PARO_ERR_INVALID, "null plan");
  paro_ctx* ctx = p->ctx;
  paro_status_t s = check_ctx(ctx);
  if (s != PARO_OK) return s;
  if (p->pl->opt.params_only) return fail(PARO_ERR_STATE, "frozen-parameter plan has no gradients or optimizer state");
  if (ctx->mode == MODE_PLANNER) return fail(PARO_ERR_STATE, "planning-only context");
  if (p->pl->opt.grad_slots > 0)
    return fail(PARO_ERR_STATE, "plan has grad_slots: gradients are produced per bucket by paro_step_streamed");
  if (!is_local(p, rank)) return fail(PARO_ERR_INVALID, "rank is not local to this process");
  uint16_t* g = reinterpret_cast<uint16_t*>(data_ptr(p, rank, BUF_GRAD, 0));
  const Planner& pl = *p->pl;
  const uint64_t key = synth_key(seed, kTagGrad, (uint64_t)rank, (uint64_t)step);
  if (pl.opt.groups.empty()) {   // dense layout: one launch, zero past psi
    CK(launch_synth_grad(g, pl.psi, pl.psi_pad, key, ctx->main));
  } else {                       // layer-aligned buckets: zero on every bucket's padded tail
    for (size_t b = 0; b < pl.buckets.size(); ++b)
      CK(launch_synth_grad_range(g + pl.buckets[b].first, pl.buckets[b].first, pl.buckets[b].second,
                                 pl.bucket_real_end[b], key, ctx->main));
  }
  CK(cudaStreamSynchronize(ctx->main));
  return PARO_OK;
}

namespace {
// Gradient source of a streamed step (grad_slots > 0): producer(user, ...) or
// the library's synthetic gradients (paro_synth hash, seed / grad_step).
struct GradSource {
  paro_grad_producer_t fn = nullptr;
  void* user = nullptr;
  uint64_t seed = 0;
  int64_t gstep = 0;
};
paro_status_t step_impl(PlanT* p, const void* const* grads, void* const* params, const paro_opt_state_t* opt_state,
                        float lr, int64_t step, const GradSource* src);
}  // namespace

paro_status_t paro_set_param_consumer(paro_plan_t p, paro_param_consumer_t consumer, void* user) {
  if (!p) return fail(PARO_ERR_INVALID, "null plan");
  if (p->ctx->mode == MODE_PLANNER) return fail(PARO_ERR_STATE, "planning-only context");
  if (p->pl->opt.params_only) return fail(PARO_ERR_STATE, "frozen-parameter plan has no step");
  p->cons_fn = consumer;
  p->cons_user = user;
  return PARO_OK;
}

paro_status_t paro_step(paro_plan_t p, const void* const* grads, void* const* params,
                        const paro_opt_state_t* opt_state, float lr, int64_t step) {
  if (!p) return fail(PARO_ERR_INVALID, "null plan");
  if (p->pl->opt.grad_slots > 0)
    return fail(PARO_ERR_STATE, "plan has grad_slots: its gradients stream in through paro_step_streamed");
  return step_impl(p, grads, params, opt_state, lr, step, nullptr);
}

paro_status_t paro_step_streamed(paro_plan_t p, paro_grad_producer_t producer, void* user, uint64_t seed,
                                 int64_t grad_step, void* const* params, const paro_opt_state_t* opt_state,
                                 float lr, int64_t step) {
  if (!p) return fail(PARO_ERR_INVALID, "null plan");
  if (p->pl->opt.grad_slots <= 0) return fail(PARO_ERR_STATE, "plan was created without grad_slots");
  GradSource src;
  src.fn = producer;
  src.user = user;
  src.seed = seed;
  src.gstep = grad_step;
  return step_impl(p, nullptr, params, opt_state, lr, step, &src);
}

namespace {
paro_status_t step_impl(PlanT* p, const void* const* grads, void* const* params, const paro_opt_state_t* opt_state,
                        float lr, int64_t step, const GradSource* src) {
  paro_ctx* ctx = p->ctx;
  paro_status_t s = check_ctx(ctx);
  if (s != PARO_OK) return s;
  if (ctx->mode == MODE_PLANNER) return fail(PARO_ERR_STATE, "planning-only context cannot step");
  if (p->pl->opt.params_only) return fail(PARO_ERR_STATE, "frozen-parameter plan has no gradients or optimizer state");
  if (step < 1) return fail(PARO_ERR_INVALID, "step must be >= 1");
  if (!opt_state) return fail(PARO_ERR_INVALID, "null opt_state");
  const Planner& pl = *p->pl;
  const int nl = (int)p->local.size();
  const int np = (int)pl.param_sizes.size();
  for (int i = 0; i < nl && pl.os_numel > 0; ++i)   // an empty model (psi = 0) has no state
    if (!opt_state[i].master || !opt_state[i].m || !opt_state[i].v)
      return fail(PARO_ERR_INVALID, "null opt_state array");
  if (grads) {
    for (int i = 0; i < nl * np; ++i)
      if (!grads[i] && pl.param_sizes[i % np] > 0) return fail(PARO_ERR_INVALID, "null gradient pointer");
  }
  // after paro_accumulate the step consumes the accumulator (R27)
  const int64_t n_acc = p->acc_count;
  if (n_acc > 0 && grads) return fail(PARO_ERR_INVALID, "grads must be NULL after paro_accumulate");
  const std::vector<DevLaunch>& red = n_acc > 0 ? p->red_acc : p->red;
  cudaStream_t S = p->opts.stream ? static_cast<cudaStream_t>(p->opts.stream) : ctx->main;
  int launches = 0;
  NvtxRange nr_step("paro_step %s t=%lld", pl.code.c_str(), (long long)step);

  // ---- host scalars of canonical Adam (double, rounded once: R6)
  const double b1 = p->opts.beta1, b2 = p->opts.beta2, dlr = lr;
  AdamArgs aa{};
  aa.alpha = p->alpha;
  aa.b1 = (float)b1;
  aa.omb1 = (float)(1.0 - b1);
  aa.b2 = (float)b2;
  aa.omb2 = (float)(1.0 - b2);
  aa.step_size = (float)(dlr / (1.0 - std::pow(b1, (double)step)));
  aa.bc2s = (float)std::sqrt(1.0 - std::pow(b2, (double)step));
  aa.eps = p->opts.eps;
  aa.has_wd = p->opts.weight_decay != 0.0f;
  aa.decay = (float)(1.0 - dlr * (double)p->opts.weight_decay);
  // unscale (R4), the mini-batch mean over accumulated micro-batches (R27) and,
  // without pre-division, the rank average (reading A4): rounded once
  const double sg_base = 1.0 / ((double)p->opts.loss_scale * (double)(n_acc > 0 ? n_acc : 1) *
                                (pl.opt.predivide ? 1.0 : (double)pl.N));
  aa.s_g = (float)sg_base;
  aa.nonfinite = p->d_nonfinite;
  aa.moved = ctx->mode == MODE_REAL ? p->d_moved : nullptr;

  CK(cudaMemsetAsync(p->d_moved, 0, 2 * sizeof(unsigned long long), S));   // moved bytes of this step
  p->moved_host[0] = p->moved_host[1] = 0;
  CK(cudaEventRecord(p->ev_fork, S));
  CK(cudaStreamWaitEvent(ctx->comm, p->ev_fork, 0));
  CK(cudaStreamWaitEvent(ctx->comp, p->ev_fork, 0));
  if (src) CK(cudaStreamWaitEvent(ctx->dma, p->ev_fork, 0));

  // ---- pack (per-parameter gradients -> flat gradient buffer)
  if (grads) {
    paro_status_t sp = pack_grads(p, grads, &launches);
    if (sp != PARO_OK) return sp;
  }
  CK(cudaMemsetAsync(p->d_nonfinite, 0, sizeof(int), ctx->comp));
  CK(cudaMemsetAsync(p->d_partials, 0, sizeof(double) * p->partials_cap, ctx->comp));
  // fused parameter all-gather: Adam stores into peers' parameter buffers, so
  // every peer must have entered this step (its reads of last step's
  // parameters are stream-ordered before it) before the first update
  // (also before copy-engine reads of the peers' raw gradient chunks)
  const bool pre_on = !p->red_pre.empty() && n_acc == 0;
  if ((!pl.sched.empty() && !pl.sched[0].param_push.empty()) || pre_on) {
    paro_status_t s0 = all_peer_barrier(p, &launches);
    if (s0 != PARO_OK) return s0;
  }

  const int nb = (int)pl.buckets.size();
  const int grid = adam_grid();
  int n_adam = 0;
  // two-phase step (clipping / non-finite skip, R28): phase 1 reduces every
  // bucket and takes the norm, the clip scale is formed on the device, phase 2
  // updates (Adam reads the scale and the skip flag from device memory)
  const bool two = pl.opt.two_phase;
  aa.s_g_dev = two ? p->d_sg : nullptr;
  aa.skip = two ? p->d_skip : nullptr;
  auto adam_bucket = [&](int b0, int b1, bool norm_only = false) -> paro_status_t {
    // one Adam (or phase-1 norm) launch over buckets [b0, b1) and every local rank
    if (b0 >= b1) return PARO_OK;   // empty model
    NvtxRange nr(norm_only ? "paro norm b%d-%d" : "paro adam b%d-%d", b0, b1 - 1);
    aa.nseg = 0;
    for (int li = 0; li < nl; ++li) {
      const int r = p->local[li];
      const int j = r / pl.M;
      const bool uniq = (pl.OS == LV_G) || (pl.OS == LV_I && j == 0) || (pl.OS == LV_N && r == 0);
      const BucketSchedule& S0 = pl.sched[b0];
      int64_t len = 0;
      for (int b = b0; b < b1; ++b) len += pl.sched[b].os_len;
      AdamSeg& sg = aa.seg[aa.nseg++];
      const std::vector<Ref>& gin = (n_acc > 0) ? S0.ghat_in_acc[r] : S0.ghat_in[r];
      sg.gnin = (int)gin.size();
      sg.graw = 0;
      sg.gf32 = 0;
      sg.gpeer = sg.ginter = sg.pinter = 0;
      sg.gwide = pl.opt.wire == 4 ? 1 : 0;
      for (int i = 0; i < sg.gnin; ++i) {
        const Ref& x = gin[i];
        sg.gin[i] = reinterpret_cast<const uint16_t*>(data_ptr(p, x.rank, x.kind, x.off));
        if (x.is_raw()) sg.graw |= 1u << i;
        else if (pl.esz[x.kind] == 4) sg.gf32 |= 1u << i;
        if (x.rank != r) {
          sg.gpeer |= 1u << i;
          if (x.rank / pl.M != r / pl.M) sg.ginter |= 1u << i;
        }
      }
      sg.master = opt_state[li].master + S0.os_off[r];
      sg.m = opt_state[li].m + S0.os_off[r];
      sg.v = opt_state[li].v + S0.os_off[r];
      sg.param = reinterpret_cast<uint16_t*>(data_ptr(p, S0.param[r].rank, S0.param[r].kind, S0.param[r].off));
      sg.n8 = len / 8;
      sg.in_norm = (uniq && (norm_only || !two)) ? 1 : 0;
      sg.npush = 0;
      if (!S0.param_push.empty())
        for (const Ref& x : S0.param_push[r]) {
          if (x.rank / pl.M != r / pl.M) sg.pinter |= 1u << sg.npush;
          sg.push[sg.npush++] = reinterpret_cast<uint16_t*>(data_ptr(p, x.rank, x.kind, x.off));
        }
    }
    aa.partials = p->d_partials + (int64_t)n_adam * grid;
    if (norm_only) {
      CK(launch_grad_norm(aa, grid, ctx->comp));
      ++n_adam;
      ++launches;
      return PARO_OK;
    }
    int64_t elems = 0, hbm = 0;
    for (int i = 0; i < aa.nseg; ++i) {
      elems += 8 * aa.seg[i].n8;
      // master/m/v read + written (24 B), bf16 parameter written (2 B), every
      // g_hat input read once (2 B each, 4 on the fp32 wire: local, or by
      // symmetry served to a peer), every fused-gather push (2 B: by symmetry,
      // a peer's push lands here)
      int gb = 0;
      for (int k = 0; k < aa.seg[i].gnin; ++k) gb += ((aa.seg[i].gf32 >> k) & 1u) ? 4 : 2;
      hbm += 8 * aa.seg[i].n8 * (26 + gb + 2 * aa.seg[i].npush);
    }
    const int pk = prof_begin(p, ctx->comp, 0, elems, hbm);
    // TMA-pipelined Adam (bulk copies also pull the fused hop's NVLink-peer
    // inputs: tools/tma_peer_test.cu measured 782 GB/s); LSU kernel on request.
    // while collectives run beside it (real N > 1) Adam keeps ~120 KB of shared
    // memory per SM so the TMA collective kernel (<= 96 KB) fits on the same SM
    // (no collective rounds beside it, e.g. everything fused: the full budget)
    bool corun = false;
    if (ctx->mode == MODE_REAL && pl.N > 1)
      for (size_t b = 0; b < p->red.size() && !corun; ++b)
        corun = red[b].nrounds > 0 || p->gat[b].nrounds > 0;
    // stores: bulk copies out of shared memory win when Adam has the GPU to itself
    // and no NVLink operands (N = 1: 0.97 of the HBM peak vs 0.90, profiles/r01);
    // beside collectives / with peer traffic the thread stores are faster
    // (real N > 1: also for the fused all-reduce when nothing runs beside Adam
    // and it pushes nothing to peers, i.e. 2x1: NNN 35.6 -> 34.0 ms,
    // profiles/r01/sweep_adam_store_fused_2x1.jsonl; with fused-gather pushes
    // (IIG 2x1 20.0 vs 20.6 ms) or a fused final hop only (GGG 2x1 17.2-17.8
    // vs 17.8-18.7 ms) the thread stores stay faster)
    bool pushes = false;
    for (int i = 0; i < aa.nseg; ++i) pushes = pushes || aa.seg[i].npush > 0;
    const int ai = p->opts.adam_impl;
    const bool tma_store = ai == 2 || ai == 4 || (ai == 0 && (pl.N == 1 || ctx->mode == MODE_EMU ||
                                                                (pl.fused_allreduce && !corun && !pushes)));
    // shared memory: the stage count follows a budget of ~120 KB while
    // collectives co-run (200 KB alone); the hard limit is what the SM has left
    // beside the largest co-running TMA rounds CTA (4 stages x 8 KB per input,
    // 228 KB per SM, 1 KB reserved per CTA).  adam_smem_kb > 0 forces both
    // (emulated / N = 1 runs of the co-run configurations).
    int budget = corun ? 120 : 200, hard = 220;
    if (corun && p->opts.comm_impl != 1) {
      int mx = 1;
      for (size_t b = 0; b < red.size(); ++b) {
        if (red[b].nrounds > 0) mx = std::max(mx, red[b].max_in);
        if (p->gat[b].nrounds > 0) mx = std::max(mx, p->gat[b].max_in);
      }
      hard = 226 - 1 - rounds_tma_smem_kb(mx);
    }
    if (p->opts.adam_smem_kb > 0) budget = hard = p->opts.adam_smem_kb;
    if (ai != 1) {
      CK(launch_adam_tma(aa, ctx->sm_count, ctx->comp, budget, tma_store ? 1 : 0, hard, &p->adam_variant,
                         &p->adam_stages, ai == 4 ? 1 : (ai == 2 ? 0 : -1)));
    } else {
      CK(launch_adam(aa, grid, ctx->comp, corun ? 1 : 0));
      p->adam_variant = ADAM_LSU;
      p->adam_stages = 0;
    }
    prof_end(p, ctx->comp, pk);
    ++n_adam;
    ++launches;
    return PARO_OK;
  };

  // grad norm: ordered fp64 finalize, then scalar all-reduces (R8, R23)
  auto norm_reduce = [&]() -> paro_status_t {
    CK(launch_norm_finalize(p->d_partials, n_adam * grid, p->d_norm, ctx->comp));
    ++launches;
    CK(cudaEventRecord(p->ev_comp, ctx->comp));
    CK(cudaStreamWaitEvent(ctx->comm, p->ev_comp, 0));
    if (ctx->mode == MODE_REAL && pl.N > 1) {
      NK(ncclAllReduce(p->d_norm, p->d_norm, 1, ncclDouble, ncclSum, ctx->world, ctx->comm));
      NK(ncclAllReduce(p->d_nonfinite, p->d_nonfinite, 1, ncclInt32, ncclMax, ctx->world, ctx->comm));
      launches += 2;
    }
    return PARO_OK;
  };

  // parameter consumer (paro_set_param_consumer): bucket b's P residency handed
  // to the caller on the sink stream as soon as it is final, so e.g. its
  // device->host copy overlaps the later buckets' work (and, in a streamed
  // step, their host->device gradients: PCIe is full duplex).  With fused
  // gathers a peer's Adam writes into our parameters: a channel-3 barrier with
  // every peer (each reaches it after its own Adam of the bucket) comes first.
  auto consume = [&](int b) -> paro_status_t {
    cudaStream_t cs = ctx->sink;
    CK(cudaStreamWaitEvent(cs, p->ev_pfinal[b], 0));
    if (!pl.sched[b].param_push.empty()) {
      uint64_t peers = 0;
      for (int x = 0; x < pl.N && ctx->mode == MODE_REAL; ++x)
        if (x != ctx->rank) peers |= uint64_t(1) << x;
      paro_status_t sb = barrier2(p, peers, cs, &launches, 3);
      if (sb != PARO_OK) return sb;
    }
    for (int li = 0; li < nl; ++li) {
      const int r = p->local[li];
      int64_t b0, b1;
      pl.residency(pl.P, r, b, &b0, &b1);
      void* src = data_ptr(p, r, BUF_PARAM, pl.buckets[b].first / pl.divl(pl.P));
      p->cons_fn(p->cons_user, r, b, b0, b1, src, cs);
    }
    CK(cudaGetLastError());
    return PARO_OK;
  };
  // streamed step: bucket b's gradients go into slot b % K once every rank is
  // done reading bucket b - K from it (its reduce and, unless two-phase, the
  // Adam that may fold it): local events, then a peer barrier on the second
  // channel, on the producer stream (ctx->dma; no copy-engine launches here)
  if (pl.N == 1 && !src) {
    if (two) {
      paro_status_t s1 = adam_bucket(0, nb, true);
      if (s1 == PARO_OK) s1 = norm_reduce();
      if (s1 != PARO_OK) return s1;
      CK(launch_clip_scale(p->d_norm, p->d_nonfinite, (double)p->opts.clip_norm, sg_base,
                           p->opts.skip_nonfinite, p->d_sg, p->d_skip, ctx->comp));
      ++launches;
      n_adam = 0;   // phase 2 reuses the partial slots (its norm flags are off)
    }
    paro_status_t s2 = adam_bucket(0, nb);   // contiguous: one launch over all buckets
    if (s2 != PARO_OK) return s2;
    if (p->cons_fn) {   // every bucket final with the one launch
      for (int b = 0; b < nb; ++b) {
        CK(cudaEventRecord(p->ev_pfinal[b], ctx->comp));
        paro_status_t sc = consume(b);
        if (sc != PARO_OK) return sc;
      }
      CK(cudaEventRecord(p->ev_cons, ctx->sink));
    }
    if (!two) {
      paro_status_t s3 = norm_reduce();
      if (s3 != PARO_OK) return s3;
    }
  } else {
    const int D = std::max(1, p->opts.pipeline_depth);
    const bool nccl = pl.opt.topology == PARO_TOPO_NCCL;
    const int me = ctx->mode == MODE_REAL ? ctx->rank : 0;
    bool dma_used = false;
    // copy-engine raw-chunk copies of bucket b into landing set b % kStageSets
    // (after the step-start barrier; set reuse waits for the reduce that read it)
    auto issue_pre = [&](int b) -> paro_status_t {
      if (b >= kStageSets) CK(cudaStreamWaitEvent(ctx->dma, p->ev_red[b - kStageSets], 0));
      paro_status_t st = run_dma_launch(p, p->red_pre[b], ctx->dma, &launches);
      if (st != PARO_OK) return st;
      CK(cudaEventRecord(p->ev_pre[b], ctx->dma));
      dma_used = true;
      return PARO_OK;
    };
    if (pre_on) {
      CK(cudaEventRecord(p->ev_comm, ctx->comm));
      CK(cudaStreamWaitEvent(ctx->dma, p->ev_comm, 0));
      for (int b = 0; b < std::min(kStageSets, nb); ++b) {
        paro_status_t st = issue_pre(b);
        if (st != PARO_OK) return st;
      }
    }
    // bucket b's parameters are final on this rank once its restore ran (or its
    // Adam, when there is no gather launch); ev_pfinal[b] marks that point
    auto do_gather = [&](int b) -> paro_status_t {
      NvtxRange nr("paro gather b%d", b);
      if (p->gat[b].dma) {   // copy engines, off the comm stream: overlaps the next reductions
        CK(cudaStreamWaitEvent(ctx->dma, p->ev_adam[b], 0));
        dma_used = true;
        paro_status_t sd = run_dma_launch(p, p->gat[b], ctx->dma, &launches);
        if (sd == PARO_OK && p->cons_fn) CK(cudaEventRecord(p->ev_pfinal[b], ctx->dma));
        return sd;
      }
      CK(cudaStreamWaitEvent(ctx->comm, p->ev_adam[b], 0));
      paro_status_t s3 = PARO_OK;
      if (nccl) {
        const int k = prof_begin(p, ctx->comm, 1, 0);
        s3 = run_nccl(p, pl.sched[b].nccl_gather[ctx->rank]);
        prof_end(p, ctx->comm, k);
        if (s3 == PARO_OK && !pl.sched[b].nccl_gather[ctx->rank].empty()) ++launches;
      } else {
        s3 = run_launch(p, p->gat[b], &launches);
      }
      if (s3 == PARO_OK && p->cons_fn) CK(cudaEventRecord(p->ev_pfinal[b], ctx->comm));
      return s3;
    };
    auto produce = [&](int b) -> paro_status_t {
      cudaStream_t ps = ctx->dma;
      const int K = pl.opt.grad_slots;
      if (b >= K) {
        CK(cudaStreamWaitEvent(ps, p->ev_red[b - K], 0));
        if (!two) CK(cudaStreamWaitEvent(ps, p->ev_adam[b - K], 0));
        uint64_t peers = 0;
        for (int x = 0; x < pl.N && ctx->mode == MODE_REAL; ++x)
          if (x != ctx->rank) peers |= uint64_t(1) << x;
        paro_status_t sb = barrier2(p, peers, ps, &launches);
        if (sb != PARO_OK) return sb;
      }
      const int64_t b0 = pl.buckets[b].first, n = pl.buckets[b].second;
      for (int li = 0; li < nl; ++li) {
        const int r = p->local[li];
        void* dst = data_ptr(p, r, BUF_GRAD, int64_t(b % K) * pl.B);
        if (src->fn) {
          src->fn(src->user, r, b, b0, b0 + n, dst, ps);
        } else {
          CK(launch_synth_grad_range(static_cast<uint16_t*>(dst), b0, n, pl.bucket_real_end[b],
                                     synth_key(src->seed, kTagGrad, (uint64_t)r, (uint64_t)src->gstep), ps));
          ++launches;
        }
      }
      CK(cudaGetLastError());
      CK(cudaEventRecord(p->ev_prod[b], ps));
      CK(cudaStreamWaitEvent(ctx->comm, p->ev_prod[b], 0));
      CK(cudaStreamWaitEvent(ctx->comp, p->ev_prod[b], 0));
      return PARO_OK;
    };
    auto do_reduce = [&](int b) -> paro_status_t {
      NvtxRange nr("paro reduce b%d", b);
      if (src) {
        paro_status_t sp = produce(b);
        if (sp != PARO_OK) return sp;
      }
      if (pre_on) CK(cudaStreamWaitEvent(ctx->comm, p->ev_pre[b], 0));
      if (nccl) {
        if (red[b].nrounds > 0) {   // fp32 wire: pre-scale the bucket into fp32 first (local round)
          paro_status_t s2 = run_launch(p, red[b], &launches);
          if (s2 != PARO_OK) return s2;
        }
        const int k = prof_begin(p, ctx->comm, 1, 0);
        paro_status_t s3 = run_nccl(p, pl.sched[b].nccl_reduce[ctx->rank]);
        prof_end(p, ctx->comm, k);
        if (s3 != PARO_OK) return s3;
        ++launches;
      } else {
        bool tail = false;   // copy-engine tail: the reduction completes on the dma stream
        paro_status_t s3 = run_launch(p, red[b], &launches, &tail);
        if (s3 != PARO_OK) return s3;
        if (tail) {
          dma_used = true;
          CK(cudaEventRecord(p->ev_red[b], ctx->dma));
          CK(cudaStreamWaitEvent(ctx->comp, p->ev_red[b], 0));
          if (pre_on && b + kStageSets < nb) return issue_pre(b + kStageSets);
          return PARO_OK;
        }
      }
      CK(cudaEventRecord(p->ev_red[b], ctx->comm));
      CK(cudaStreamWaitEvent(ctx->comp, p->ev_red[b], 0));
      if (pre_on && b + kStageSets < nb) return issue_pre(b + kStageSets);
      return PARO_OK;
    };
    if (two) {
      // phase 1: every reduction (g_hat stays resident: one slot per bucket), norm per bucket
      for (int b = 0; b < nb; ++b) {
        paro_status_t s3 = do_reduce(b);
        if (s3 == PARO_OK) s3 = adam_bucket(b, b + 1, true);
        if (s3 != PARO_OK) return s3;
      }
      paro_status_t s4 = norm_reduce();
      if (s4 != PARO_OK) return s4;
      CK(cudaEventRecord(p->ev_comm, ctx->comm));
      CK(cudaStreamWaitEvent(ctx->comp, p->ev_comm, 0));
      CK(launch_clip_scale(p->d_norm, p->d_nonfinite, (double)p->opts.clip_norm, sg_base,
                           p->opts.skip_nonfinite, p->d_sg, p->d_skip, ctx->comp));
      ++launches;
      n_adam = 0;   // phase 2 reuses the partial slots (its norm flags are off)
    }
    for (int b = 0; b < nb; ++b) {
      if (!two) {
        // staging sets / g_hat slots are reused kStageSets / nslots buckets later:
        // the Adam that reads them (fused final hop) must be done first
        if (pl.nslots > 0 && b >= pl.nslots) CK(cudaStreamWaitEvent(ctx->comm, p->ev_adam[b - pl.nslots], 0));
        if (b >= kStageSets) CK(cudaStreamWaitEvent(ctx->comm, p->ev_adam[b - kStageSets], 0));
        paro_status_t s3 = do_reduce(b);
        if (s3 != PARO_OK) return s3;
      }
      paro_status_t s4 = adam_bucket(b, b + 1);
      if (s4 != PARO_OK) return s4;
      CK(cudaEventRecord(p->ev_adam[b], ctx->comp));
      if (p->cons_fn && p->gat[b].nrounds == 0 && !p->gat[b].dma && (!nccl || pl.sched[b].nccl_gather[me].empty()))
        CK(cudaEventRecord(p->ev_pfinal[b], ctx->comp));   // no restore launch: final after Adam
      if (b >= D) {
        paro_status_t s5 = do_gather(b - D);
        if (s5 != PARO_OK) return s5;
      }
    }
    for (int b = std::max(0, nb - D); b < nb; ++b) {
      paro_status_t s5 = do_gather(b);
      if (s5 != PARO_OK) return s5;
    }
    if (p->cons_fn) {   // in bucket order, each as soon as its parameters are final
      for (int b = 0; b < nb; ++b) {
        paro_status_t sc = consume(b);
        if (sc != PARO_OK) return sc;
      }
      CK(cudaEventRecord(p->ev_cons, ctx->sink));
    }
    if (dma_used) {   // the step-end barrier comes after every copy-engine transfer
      CK(cudaEventRecord(p->ev_dma, ctx->dma));
      CK(cudaStreamWaitEvent(ctx->comm, p->ev_dma, 0));
    }
    if (!two) {
      paro_status_t s6 = norm_reduce();
      if (s6 != PARO_OK) return s6;
    }
  }
  CK(cudaEventRecord(p->ev_comp, ctx->comp));
  CK(cudaStreamWaitEvent(ctx->comm, p->ev_comp, 0));
  // ---- step-end barrier with every peer
  {
    paro_status_t s6 = all_peer_barrier(p, &launches);
    if (s6 != PARO_OK) return s6;
  }
  // ---- unpack into caller parameter tensors
  if (params) {
    int k = 0;
    int64_t maxn = 0;
    CK(cudaEventSynchronize(p->ev_unpack_staged));
    PackEntry* hu = p->h_pack + p->pack_cap;
    PackEntry* du = p->d_pack + p->pack_cap;
    for (int li = 0; li < nl; ++li) {
      const int r = p->local[li];
      if (pl.P == LV_N) {
        for (int i = 0; i < np; ++i) {
          if (pl.param_sizes[i] == 0) continue;
          hu[k].src = reinterpret_cast<const uint16_t*>(data_ptr(p, r, BUF_PARAM, pl.param_offsets[i]));
          hu[k].dst = static_cast<uint16_t*>(params[li * np + i]);
          hu[k].n = pl.param_sizes[i];
          maxn = std::max(maxn, pl.param_sizes[i]);
          ++k;
        }
      } else {
        hu[k].src = reinterpret_cast<const uint16_t*>(data_ptr(p, r, BUF_PARAM, 0));
        hu[k].dst = static_cast<uint16_t*>(params[li]);
        hu[k].n = pl.p_numel;
        maxn = std::max(maxn, pl.p_numel);
        ++k;
      }
    }
    if (k > 0) {
      CK(cudaMemcpyAsync(du, hu, sizeof(PackEntry) * k, cudaMemcpyHostToDevice, ctx->comm));
      CK(cudaEventRecord(p->ev_unpack_staged, ctx->comm));
      CK(launch_pack(du, k, maxn, ctx->comm));
      ++launches;
    }
  }
  CK(cudaEventRecord(p->ev_comm, ctx->comm));
  CK(cudaStreamWaitEvent(S, p->ev_comm, 0));
  if (p->cons_fn) CK(cudaStreamWaitEvent(S, p->ev_cons, 0));   // the step includes the consumption
  p->last_stream = S;
  p->last_launches = launches;
  p->stepped = true;
  p->last_step_acc = n_acc > 0;
  p->acc_count = 0;
  if (p->prof) {
    ++p->prof_steps;
    p->prof_launches += launches;
  }
  return PARO_OK;
}

}  // namespace

paro_status_t paro_accumulate(paro_plan_t p, const void* const* grads) {
  if (!p) return fail(PARO_ERR_INVALID, "null plan");
  paro_ctx* ctx = p->ctx;
  paro_status_t s = check_ctx(ctx);
  if (s != PARO_OK) return s;
  if (ctx->mode == MODE_PLANNER) return fail(PARO_ERR_STATE, "planning-only context cannot accumulate");
  if (p->pl->opt.params_only) return fail(PARO_ERR_STATE, "frozen-parameter plan has no gradients or optimizer state");
  const Planner& pl = *p->pl;
  if (!pl.opt.accum) return fail(PARO_ERR_STATE, "plan was created without grad_accum");
  const int nl = (int)p->local.size();
  const int np = (int)pl.param_sizes.size();
  if (grads) {
    for (int i = 0; i < nl * np; ++i)
      if (!grads[i] && pl.param_sizes[i % np] > 0) return fail(PARO_ERR_INVALID, "null gradient pointer");
  }
  cudaStream_t S = p->opts.stream ? static_cast<cudaStream_t>(p->opts.stream) : ctx->main;
  int launches = 0;
  CK(cudaEventRecord(p->ev_fork, S));
  CK(cudaStreamWaitEvent(ctx->comm, p->ev_fork, 0));
  CK(cudaStreamWaitEvent(ctx->comp, p->ev_fork, 0));
  if (grads) {
    paro_status_t sp = pack_grads(p, grads, &launches);
    if (sp != PARO_OK) return sp;
  }
  const std::vector<DevLaunch>& acc = (p->acc_count == 0) ? p->acc_first : p->acc_next;
  const bool pre_on = !p->acc_pre.empty();
  if (pre_on) {   // copy-engine reads of the peers' raw chunks: every peer has its micro-batch in place
    paro_status_t s0 = all_peer_barrier(p, &launches);
    if (s0 != PARO_OK) return s0;
  }
  for (size_t b = 0; b < pl.buckets.size(); ++b) {
    if (pre_on) {   // serial on the comm stream: the landing set is reused three buckets later
      paro_status_t s2 = run_dma_launch(p, p->acc_pre[b], ctx->comm, &launches);
      if (s2 != PARO_OK) return s2;
    }
    paro_status_t s3 = run_launch(p, acc[b], &launches);
    if (s3 != PARO_OK) return s3;
  }
  {
    paro_status_t s6 = all_peer_barrier(p, &launches);   // peers are done reading our gradients
    if (s6 != PARO_OK) return s6;
  }
  CK(cudaEventRecord(p->ev_comm, ctx->comm));
  CK(cudaStreamWaitEvent(S, p->ev_comm, 0));
  p->last_stream = S;
  ++p->acc_count;
  if (p->prof) p->prof_launches += launches;
  return PARO_OK;
}

paro_status_t paro_gather_window(paro_plan_t p, int rank, int64_t bucket, int slot, void* stream, void** out) {
  if (!p || !out) return fail(PARO_ERR_INVALID, "null argument");
  paro_ctx* ctx = p->ctx;
  paro_status_t s = check_ctx(ctx);
  if (s != PARO_OK) return s;
  if (ctx->mode == MODE_PLANNER) return fail(PARO_ERR_STATE, "planning-only context");
  const Planner& pl = *p->pl;
  if (!is_local(p, rank)) return fail(PARO_ERR_INVALID, "rank is not local to this process");
  if (bucket < 0 || bucket >= (int64_t)pl.buckets.size()) return fail(PARO_ERR_INVALID, "bucket out of range");
  if (pl.P == LV_N || pl.N == 1) {   // parameters are resident: the bucket is a view of the parameter buffer
    *out = data_ptr(p, rank, BUF_PARAM, pl.buckets[bucket].first);
    return PARO_OK;
  }
  if (p->win.empty()) return fail(PARO_ERR_STATE, "plan was created without gather_windows");
  if (slot < 0 || slot >= (int)p->win.size()) return fail(PARO_ERR_INVALID, "window slot out of range");
  if (ctx->mode == MODE_EMU && rank != p->local[0])
    return fail(PARO_ERR_INVALID, "emulated mode gathers every rank at once: pass rank 0");
  cudaStream_t S = stream ? static_cast<cudaStream_t>(stream)
                          : (p->opts.stream ? static_cast<cudaStream_t>(p->opts.stream) : ctx->main);
  int launches = 0;
  CK(cudaEventRecord(p->ev_fork, S));
  CK(cudaStreamWaitEvent(ctx->comm, p->ev_fork, 0));
  paro_status_t s3 = run_launch(p, p->win[slot][bucket], &launches);
  if (s3 != PARO_OK) return s3;
  CK(cudaEventRecord(p->ev_comm, ctx->comm));
  CK(cudaStreamWaitEvent(S, p->ev_comm, 0));
  *out = data_ptr(p, rank, BUF_WIN, int64_t(slot) * pl.B);
  p->last_stream = S;
  if (p->prof) p->prof_launches += launches;
  return PARO_OK;
}

paro_status_t paro_collective(paro_plan_t p, int what) {
  if (!p) return fail(PARO_ERR_INVALID, "null plan");
  paro_ctx* ctx = p->ctx;
  paro_status_t s = check_ctx(ctx);
  if (s != PARO_OK) return s;
  if (p->pl->opt.params_only) return fail(PARO_ERR_STATE, "frozen-parameter plan has no gradients or optimizer state");
  if (ctx->mode == MODE_PLANNER) return fail(PARO_ERR_STATE, "planning-only context");
  if (what != 0 && what != 1) return fail(PARO_ERR_INVALID, "what must be 0 (reduce) or 1 (gather)");
  const Planner& pl = *p->pl;
  // a plan that folds part of its gradient reduction into the Adam kernel (the
  // inter all-reduce, R31, or the owner's final hop for OS = G) has reduce
  // launches that do not complete the reduction on their own
  if (what == 0 && pl.N > 1 && pl.opt.topology != PARO_TOPO_NCCL) {
    bool folded = pl.fused_allreduce;
    for (const BucketSchedule& S0 : pl.sched)
      for (const auto& gin : S0.ghat_in) folded = folded || gin.size() > 1;
    if (folded)
      return fail(PARO_ERR_STATE,
                  "plan folds part of its reduction into the Adam kernel (fused inter all-reduce or final hop): "
                  "paro_collective(0) needs a plan made with fuse_allreduce = 0");
  }
  cudaStream_t S = p->opts.stream ? static_cast<cudaStream_t>(p->opts.stream) : ctx->main;
  int launches = 0;
  bool tails = false;
  CK(cudaEventRecord(p->ev_fork, S));
  CK(cudaStreamWaitEvent(ctx->comm, p->ev_fork, 0));
  const bool nccl = pl.opt.topology == PARO_TOPO_NCCL;
  for (size_t b = 0; b < pl.buckets.size() && pl.N > 1; ++b) {
    if (nccl) {
      if (what == 0 && p->red[b].nrounds > 0) {   // fp32 wire: pre-scale into fp32 first
        paro_status_t s2 = run_launch(p, p->red[b], &launches);
        if (s2 != PARO_OK) return s2;
      }
      const auto& calls = what == 0 ? pl.sched[b].nccl_reduce[ctx->rank] : pl.sched[b].nccl_gather[ctx->rank];
      const int k = prof_begin(p, ctx->comm, 1, 0);
      paro_status_t s3 = run_nccl(p, calls);
      prof_end(p, ctx->comm, k);
      if (s3 != PARO_OK) return s3;
      ++launches;
    } else {
      paro_status_t s3 = run_launch(p, what == 0 ? p->red[b] : p->gat[b], &launches, &tails);
      if (s3 != PARO_OK) return s3;
    }
  }
  if (tails) {   // copy-engine tails (the later buckets' kernels ran beside them)
    CK(cudaEventRecord(p->ev_dma, ctx->dma));
    CK(cudaStreamWaitEvent(ctx->comm, p->ev_dma, 0));
  }
  CK(cudaEventRecord(p->ev_comm, ctx->comm));
  CK(cudaStreamWaitEvent(S, p->ev_comm, 0));
  p->last_stream = S;
  if (p->prof) {
    ++p->prof_steps;
    p->prof_launches += launches;
  }
  return PARO_OK;
}

paro_status_t paro_profile_start(paro_plan_t p, int max_launches) {
  if (!p) return fail(PARO_ERR_INVALID, "null plan");
  paro_ctx* ctx = p->ctx;
  paro_status_t s = check_ctx(ctx);
  if (s != PARO_OK) return s;
  if (ctx->mode == MODE_PLANNER) return fail(PARO_ERR_STATE, "planning-only context");
  if (max_launches < 1) return fail(PARO_ERR_INVALID, "max_launches must be >= 1");
  for (cudaEvent_t e : p->prof_ev) cudaEventDestroy(e);
  p->prof_ev.assign(2 * (size_t)max_launches, nullptr);
  for (auto& e : p->prof_ev) CK(cudaEventCreate(&e));
  p->prof_kind.assign(max_launches, 0);
  p->prof_amount.assign(max_launches, 0);
  p->prof_hbm.assign(max_launches, 0);
  p->prof_used = 0;
  p->prof_steps = 0;
  p->prof_launches = 0;
  if (ctx->mode == MODE_REAL && !p->d_trace) {
    CK(cudaMalloc(&p->d_trace, sizeof(uint64_t) * kTraceLaunches * ctx->sm_count * kTraceSlots));
  }
  p->trace_nrounds.clear();
  p->trace_grids.clear();
  p->prof = true;
  return PARO_OK;
}

paro_status_t paro_profile_stop(paro_plan_t p, paro_profile_t* out) {
  if (!p || !out) return fail(PARO_ERR_INVALID, "null argument");
  paro_ctx* ctx = p->ctx;
  paro_status_t s = check_ctx(ctx);
  if (s != PARO_OK) return s;
  std::memset(out, 0, sizeof(*out));
  CK(cudaDeviceSynchronize());
  for (int k = 0; k < p->prof_used; ++k) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, p->prof_ev[2 * k], p->prof_ev[2 * k + 1]));
    if (p->prof_kind[k] == 0) {
      out->adam_ms += ms;
      out->adam_launches += 1;
      out->adam_elems += p->prof_amount[k];
      out->adam_hbm_bytes += p->prof_hbm[k];
    } else {
      out->comm_ms += ms;
      out->comm_launches += 1;
      out->comm_bytes += p->prof_amount[k];
      out->comm_hbm_bytes += p->prof_hbm[k];
    }
  }
  out->steps = p->prof_steps;
  out->kernel_launches = p->prof_launches;
  out->adam_variant = p->adam_variant;
  out->adam_stages = p->adam_stages;
  // device-side trace of the first collective launches: where the time goes
  if (!p->trace_nrounds.empty()) {
    const int S = p->ctx->sm_count;
    std::vector<uint64_t> tr((size_t)p->trace_nrounds.size() * S * kTraceSlots);
    CK(cudaMemcpy(tr.data(), p->d_trace, tr.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    double bar = 0, work = 0, fin = 0;
    for (size_t l = 0; l < p->trace_nrounds.size(); ++l) {
      const uint64_t* t = tr.data() + l * S * kTraceSlots;
      const int G = p->trace_grids[l];
      auto mx = [&](int slot) { uint64_t m = 0; for (int b = 0; b < G; ++b) m = std::max(m, t[b * kTraceSlots + slot]); return m; };
      auto mn = [&](int slot) { uint64_t m = ~0ull; for (int b = 0; b < G; ++b) m = std::min(m, t[b * kTraceSlots + slot]); return m; };
      uint64_t prev = mn(0);
      const int R = std::min(p->trace_nrounds[l], (kTraceSlots - 2) / 2);
      const bool dump = std::getenv("PARO_TRACE_DUMP") != nullptr;
      if (dump) std::fprintf(stderr, "[paro trace] rank %d launch %zu: cta start spread %.2f us", p->ctx->rank, l,
                             1e-3 * (double)(mx(0) - mn(0)));
      for (int r = 0; r < R; ++r) {
        const uint64_t be = mx(1 + 2 * r), we = mx(2 + 2 * r);
        bar += (double)(be - prev);
        work += (double)(we - be);
        if (dump) std::fprintf(stderr, " | r%d bar %.2f work %.2f", r, 1e-3 * (double)(be - prev), 1e-3 * (double)(we - be));
        prev = we;
      }
      if (dump) std::fprintf(stderr, " | end %.2f\n", 1e-3 * (double)(mx(kTraceSlots - 1) - prev));
      fin += (double)(mx(kTraceSlots - 1) - prev);
    }
    out->traced_launches = (int64_t)p->trace_nrounds.size();
    out->traced_barrier_ms = bar * 1e-6;
    out->traced_work_ms = work * 1e-6;
    out->traced_final_ms = fin * 1e-6;
  }
  p->prof = false;
  for (cudaEvent_t e : p->prof_ev) cudaEventDestroy(e);
  p->prof_ev.clear();
  p->prof_used = 0;
  return PARO_OK;
}

paro_status_t paro_step_stats(paro_plan_t p, paro_step_stats_t* out) {
  if (!p || !out) return fail(PARO_ERR_INVALID, "null argument");
  paro_ctx* ctx = p->ctx;
  paro_status_t s = check_ctx(ctx);
  if (s != PARO_OK) return s;
  if (ctx->mode == MODE_PLANNER) return fail(PARO_ERR_STATE, "planning-only context");
  std::memset(out, 0, sizeof(*out));
  if (!p->stepped) return fail(PARO_ERR_STATE, "no step has run on this plan");
  {
    paro_status_t sw = sync_watch(ctx, p->last_stream);
    if (sw != PARO_OK) return sw;
  }
  for (char* r : p->region) {
    int err = 0;
    CK(cudaMemcpy(&err, r + 520, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) {
      ctx->sticky = PARO_ERR_TIMEOUT;
      ctx->sticky_msg = "a cross-GPU wait timed out on the device (peer never arrived)";
      return fail(PARO_ERR_TIMEOUT, ctx->sticky_msg);
    }
  }
  double nsq = 0;
  int nf = 0;
  CK(cudaMemcpy(&nsq, p->d_norm, sizeof(double), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&nf, p->d_nonfinite, sizeof(int), cudaMemcpyDeviceToHost));
  out->grad_norm = std::sqrt(nsq);
  out->nonfinite = nf;
  const int me = ctx->mode == MODE_REAL ? ctx->rank : 0;
  out->sent_intra = p->last_step_acc ? p->pl->accstep_send_intra[me] : p->pl->send_intra[me];
  out->sent_inter = p->last_step_acc ? p->pl->accstep_send_inter[me] : p->pl->send_inter[me];
  out->kernel_launches = p->last_launches;
  out->moved_intra = out->moved_inter = -1;
  if (ctx->mode == MODE_REAL && p->pl->opt.topology != PARO_TOPO_NCCL) {
    unsigned long long mv[2] = {0, 0};
    CK(cudaMemcpy(mv, p->d_moved, sizeof(mv), cudaMemcpyDeviceToHost));
    out->moved_intra = (int64_t)mv[0] + p->moved_host[0];
    out->moved_inter = (int64_t)mv[1] + p->moved_host[1];
  }
  return PARO_OK;
}

paro_status_t paro_plan_destroy(paro_plan_t p) {
  destroy_plan(p);
  return PARO_OK;
}

}  // extern "C"
