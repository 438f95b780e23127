// planner.cpp — see planner.h.  Host only.
//
// Schedules are written in the pull model used by the sm_100a kernels: in a
// round, a rank READS its ring predecessor's partial (over NVLink in real
// mode) and writes its own result locally.  The arithmetic each element sees
// is exactly the ring of the paper in canonical order R2:
// the chain for block c starts at member c+1 and ends at its owner c.
#include "planner.h"

#include <algorithm>
#include <cstdlib>
#include <functional>
#include <stdexcept>

namespace paro {

namespace {

constexpr int64_t kQuantum = 64;      // elements per shard granule (R21)
constexpr int64_t kAlignElems = 128;  // 256-byte alignment of buffer kinds
constexpr int64_t kOneRoundExtraBytes = int64_t(6) << 20;   // one-shot AR: extra bytes worth one barrier
constexpr int64_t kOneShotMaxBytes = int64_t(256) << 20;    // one-shot topology: larger buckets use HO-Ring

// PARO_ONESHOT_MAX_MB overrides the threshold (measurement runs)
int64_t oneshot_max_bytes() {
  const char* v = std::getenv("PARO_ONESHOT_MAX_MB");
  return v ? int64_t(std::atoll(v)) << 20 : kOneShotMaxBytes;
}

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

Ref at(Ref r, int64_t d) {
  r.off += d;
  return r;
}

struct Piece {
  int64_t src_off;  // offset in the contribution's address space
  int64_t len;
  int64_t blk_off;  // offset inside the dense block (stage / dest space)
};

using PieceFn = std::function<std::vector<Piece>(int c)>;
using ContribFn = std::function<Ref(int q, int c, const Piece& pc)>;
using BaseFn = std::function<Ref(int q, int slot)>;

struct FinalIn {   // inputs of a ring RS's final hop at member q, per piece
  std::vector<Piece> pieces;
  std::vector<Ref> pin;   // partial from the predecessor (rank == -1: none, k == 1)
  std::vector<Ref> own;   // own contribution
};

Task make_task(int64_t n, std::initializer_list<Ref> ins, Ref dst) {
  Task t;
  t.n = n;
  t.nin = 0;
  for (const Ref& r : ins) {
    if (r.rank < 0) continue;
    t.in[t.nin++] = r;
  }
  t.dst = dst;
  return t;
}

// Ring reduce-scatter body over `ranks` (k members).
//  pull: member q READS its predecessor's partial (or raw contribution at the
//        first hop) and writes locally; non-final hops at round0 + t, t <= k-3;
//        the final hop may run from round0 + k - 2.
//  push: member q combines the partial its predecessor WROTE into q's stage
//        with its own contribution and STORES the result into its successor's
//        stage; hops at round0 + t, t <= k-2; the final (local) fold may run
//        from round0 + k - 1.
// Either way block c's chain is c+1, c+2, ..., c (canonical order R2).
struct RingBody {
  std::vector<FinalIn> fin;
  int final_off = 0;   // earliest final-fold round, relative to round0
};

RingBody ring_rs_body(Launch& L, bool push, const std::vector<int>& ranks, const PieceFn& pieces,
                      const ContribFn& contrib, const BaseFn& stage, int round0) {
  const int k = (int)ranks.size();
  RingBody rb;
  rb.fin.resize(k);
  if (k == 1) {
    rb.fin[0].pieces = pieces(0);
    for (const Piece& pc : rb.fin[0].pieces) {
      rb.fin[0].pin.push_back(Ref{});
      rb.fin[0].own.push_back(contrib(0, 0, pc));
    }
    rb.final_off = 0;
    return rb;
  }
  if (!push) {
    for (int t = 0; t + 2 < k; ++t) {
      for (int q = 0; q < k; ++q) {
        const int c = ((q - t - 2) % k + k) % k;
        const int pred = (q - 1 + k) % k;
        for (const Piece& pc : pieces(c)) {
          Ref in0 = (t == 0) ? contrib(pred, c, pc) : at(stage(pred, (t - 1) % 2), pc.blk_off);
          L.add(round0 + t, ranks[q], make_task(pc.len, {in0, contrib(q, c, pc)}, at(stage(q, t % 2), pc.blk_off)));
        }
      }
    }
    for (int q = 0; q < k; ++q) {
      const int pred = (q - 1 + k) % k;
      rb.fin[q].pieces = pieces(q);
      for (const Piece& pc : rb.fin[q].pieces) {
        rb.fin[q].pin.push_back(k == 2 ? contrib(pred, q, pc) : at(stage(pred, (k - 3) % 2), pc.blk_off));
        rb.fin[q].own.push_back(contrib(q, q, pc));
      }
    }
    rb.final_off = k - 2;
    return rb;
  }
  for (int t = 0; t + 1 < k; ++t) {
    for (int q = 0; q < k; ++q) {
      const int c = ((q - 1 - t) % k + k) % k;
      const int succ = (q + 1) % k;
      for (const Piece& pc : pieces(c)) {
        Ref d = at(stage(succ, t % 2), pc.blk_off);
        if (t == 0) L.add(round0, ranks[q], make_task(pc.len, {contrib(q, c, pc)}, d));
        else L.add(round0 + t, ranks[q], make_task(pc.len, {at(stage(q, (t - 1) % 2), pc.blk_off), contrib(q, c, pc)}, d));
      }
    }
  }
  for (int q = 0; q < k; ++q) {
    rb.fin[q].pieces = pieces(q);
    for (const Piece& pc : rb.fin[q].pieces) {
      rb.fin[q].pin.push_back(at(stage(q, (k - 2) % 2), pc.blk_off));
      rb.fin[q].own.push_back(contrib(q, q, pc));
    }
  }
  rb.final_off = k - 1;
  return rb;
}

// Plain ring RS: body + final fold into dest(q) (block space).  Returns rounds used.
int ring_rs(Launch& L, bool push, const std::vector<int>& ranks, const PieceFn& pieces,
            const ContribFn& contrib, const BaseFn& stage, const std::function<Ref(int q)>& dest, int round0) {
  const int k = (int)ranks.size();
  RingBody rb = ring_rs_body(L, push, ranks, pieces, contrib, stage, round0);
  bool any = false;
  for (int q = 0; q < k; ++q) {
    for (size_t i = 0; i < rb.fin[q].pieces.size(); ++i) {
      const Piece& pc = rb.fin[q].pieces[i];
      Ref d = at(dest(q), pc.blk_off);
      const Ref& own = rb.fin[q].own[i];
      if (k == 1 && own.rank == d.rank && own.kind == d.kind && own.off == d.off) continue;
      L.add(round0 + rb.final_off, ranks[q], make_task(pc.len, {rb.fin[q].pin[i], own}, d));
      any = true;
    }
  }
  return (k == 1 && !any) ? 0 : rb.final_off + 1;
}

// Ring all-gather in place: member q owns block q in base(q).
//  pull: round t, q copies block (q-1-t) from its predecessor;
//  push: round t, q stores block (q-t) into its successor.  Returns k - 1.
int ring_ag(Launch& L, bool push, const std::vector<int>& ranks, const PieceFn& pieces,
            const std::function<Ref(int q)>& base, int round0) {
  const int k = (int)ranks.size();
  for (int t = 0; t + 1 < k; ++t) {
    for (int q = 0; q < k; ++q) {
      if (!push) {
        const int c = ((q - 1 - t) % k + k) % k;
        const int pred = (q - 1 + k) % k;
        for (const Piece& pc : pieces(c))
          L.add(round0 + t, ranks[q], make_task(pc.len, {at(base(pred), pc.src_off)}, at(base(q), pc.src_off)));
      } else {
        const int c = ((q - t) % k + k) % k;
        const int succ = (q + 1) % k;
        for (const Piece& pc : pieces(c))
          L.add(round0 + t, ranks[q], make_task(pc.len, {at(base(q), pc.src_off)}, at(base(succ), pc.src_off)));
      }
    }
  }
  return k - 1;
}

}  // namespace

// ----------------------------------------------------------------- Launch
void Launch::add(int round, int rank, const Task& t) {
  if ((int)rounds.size() <= round) rounds.resize(round + 1, std::vector<std::vector<Task>>(n_ranks));
  rounds[round][rank].push_back(t);
}

std::vector<int> Launch::reads(int r, int rank) const {
  // every other rank whose memory `rank` reads (pull) or writes (push) in round r
  std::vector<int> out;
  if (r < 0 || r >= (int)rounds.size()) return out;
  auto add = [&](int x) {
    if (x != rank && std::find(out.begin(), out.end(), x) == out.end()) out.push_back(x);
  };
  for (const Task& t : rounds[r][rank]) {
    for (int i = 0; i < t.nin; ++i) add(t.in[i].rank);
    add(t.dst.rank);
  }
  return out;
}

uint64_t Launch::barrier_peers(int r, int rank) const {
  uint64_t m = 0;
  if (r >= (int)rounds.size() && !final_extra.empty()) m |= final_extra[rank];
  if (r == 0 && !first_extra.empty()) m |= first_extra[rank];
  for (int rr = r - 1; rr <= r; ++rr) {
    if (rr < 0 || rr >= (int)rounds.size()) continue;
    for (int x : reads(rr, rank)) m |= uint64_t(1) << x;
    for (int x = 0; x < n_ranks; ++x) {
      if (x == rank) continue;
      auto rx = reads(rr, x);
      if (std::find(rx.begin(), rx.end(), rank) != rx.end()) m |= uint64_t(1) << x;
    }
  }
  return m;
}

// ----------------------------------------------------------------- validation
Level parse_level(char c) {
  if (c == 'N') return LV_N;
  if (c == 'I') return LV_I;
  if (c == 'G') return LV_G;
  throw std::invalid_argument("bad level");
}

std::string validate_strategy(const std::string& code) {
  if (code.size() != 3) return "strategy code must have 3 characters";
  for (int i = 0; i < 3; ++i) {
    char c = code[i];
    if (c != 'N' && c != 'I' && c != 'G')
      return std::string("invalid shard level '") + c + "' at position " + std::to_string(i + 1);
  }
  // Principle 1: OS at least as finely sharded as P and G.
  Level p = parse_level(code[0]), g = parse_level(code[1]), o = parse_level(code[2]);
  if (o < p || o < g)
    return "strategy '" + code + "' violates Principle 1 (S_P>=S_OS and S_G>=S_OS)";
  return "";
}

std::string validate_cluster(int N, int M) {
  if (N < 1 || M < 1) return "n_gpus and group_size must be >= 1";
  if (N > 64) return "n_gpus must be <= 64";
  if (N % M != 0) return "group_size must divide n_gpus";
  return "";
}

// ----------------------------------------------------------------- Planner
Planner::Planner(int N_, int M_, const std::string& code_, const std::vector<int64_t>& sizes,
                 const PlanOptions& opt_)
    : N(N_), M(M_), g(0), code(code_), opt(opt_), param_sizes(sizes) {
  std::string e = validate_cluster(N, M);
  if (!e.empty()) throw std::invalid_argument(e);
  e = validate_strategy(code);
  if (!e.empty()) throw std::invalid_argument(e);
  g = N / M;
  P = parse_level(code[0]);
  G = parse_level(code[1]);
  OS = parse_level(code[2]);
  // Degenerate splits: with M == 1 a group is one GPU (I == N); with g == 1 a
  // group is the world (I == G).  Same residencies, same bits, no copy rounds.
  auto norm = [&](Level l) {
    if (l == LV_I && M == 1) return LV_N;
    if (l == LV_I && g == 1) return LV_G;
    return l;
  };
  P = norm(P);
  G = norm(G);
  OS = norm(OS);
  for (int64_t s : sizes)
    if (s < 0) throw std::invalid_argument("param sizes must be >= 0");
  if (opt.topology < 0 || opt.topology > 6) throw std::invalid_argument("unknown topology");
  if (opt.topology == 6 && N > kMaxIn - 1)
    throw std::invalid_argument("one-shot topology needs n_gpus <= 15");
  if (opt.topology == 6 && opt.push) throw std::invalid_argument("one-shot topology is pull-only (transport = pull)");
  if (opt.topology == 3 && (M > kMaxIn || g > kMaxIn))
    throw std::invalid_argument("direct topology needs group_size and n_groups <= 16");
  if (opt.pipeline_depth < 1) opt.pipeline_depth = 1;
  if (opt.accum && opt.topology == 4)
    throw std::invalid_argument("gradient accumulation is not available with the NCCL comparator topology");
  if (opt.accum && opt.topology == 3 && (M >= kMaxIn || g >= kMaxIn))
    throw std::invalid_argument("gradient accumulation with the direct topology needs group_size and n_groups < 16");
  if (opt.params_only) opt.accum = opt.two_phase = opt.ce_reduce = false;
  if (opt.grad_slots < 0) throw std::invalid_argument("grad_slots must be >= 0");
  if (opt.grad_slots > 0 && (opt.accum || opt.ce_reduce))
    throw std::invalid_argument("grad_slots cannot be combined with grad_accum or copy_engine = 2");
  if (opt.wire != 2 && opt.wire != 4) throw std::invalid_argument("wire_dtype must be 0 (bf16) or 1 (fp32)");
  if (opt.wire == 4 && opt.ce_reduce)
    throw std::invalid_argument("wire_dtype = 1 (fp32) is not available with copy_engine = 2");
  layout();
  if (N == 1 && opt.two_phase && opt.grad_slots > 0 && opt.grad_slots < (int64_t)buckets.size())
    throw std::invalid_argument(
        "a two-phase step (clip_norm / skip_nonfinite) at N = 1 updates from the raw gradients after the norm "
        "pass: grad_slots must be 0 or >= the number of buckets");
  build_schedule();
  if (opt.params_only) {   // keep only the forward/backward parameter gathers
    for (BucketSchedule& S : sched) {
      BucketSchedule w;
      w.window = S.window;
      w.nccl_reduce.assign(N, {});
      w.nccl_gather.assign(N, {});
      w.ghat.assign(N, Ref{});
      w.ghat_in.assign(N, {});
      w.param = std::vector<Ref>(N, Ref{0, BUF_PARAM, 0});
      w.os_off.assign(N, 0);
      w.os_len = 0;
      S = w;
    }
    grad_ops.clear();
    rest_ops.clear();
  }
  validate_refs();
  count_bytes();
}

void Planner::residency(Level l, int r, int64_t b, int64_t* begin, int64_t* end) const {
  const int64_t s = buckets[b].first, n = buckets[b].second;
  const int j = grp(r), p = pos(r);
  if (l == LV_N) {
    *begin = s;
    *end = s + n;
  } else if (l == LV_I) {
    const int64_t c = n / M;
    *begin = s + p * c;
    *end = *begin + c;
  } else {
    const int64_t c = n / N;
    *begin = s + int64_t(seg(j, p)) * c;
    *end = *begin + c;
  }
}

int64_t Planner::mem_bytes(int state) const {
  if (state == 0) return 2 * p_numel;
  if (opt.params_only && state != 0) return 0;
  if (state == 1) return G == LV_N ? 2 * psi_pad : int64_t(opt.wire) * g_numel;
  return 12 * os_numel;
}

void Planner::layout() {
  const int64_t unit = int64_t(N) * kQuantum;
  psi = 0;
  param_offsets.clear();
  buckets.clear();
  bucket_real_end.clear();
  if (!opt.groups.empty()) {
    // layer-aligned buckets (NEXT-2): bucket k = tensors [groups[k], groups[k+1]),
    // dense, zero-padded at its end to a multiple of N*64 (R21 per bucket)
    const int n = (int)param_sizes.size();
    const std::vector<int64_t>& gs = opt.groups;
    bool ok = gs[0] == 0 && gs.back() < std::max(n, 1);
    for (size_t k = 1; k < gs.size(); ++k) ok = ok && gs[k] > gs[k - 1];
    if (!ok) throw std::invalid_argument("bucket groups must start at tensor 0 and increase strictly below n_params");
    int64_t o = 0;
    for (size_t k = 0; k < gs.size(); ++k) {
      const int64_t start = o;
      const int64_t t1 = (k + 1 < gs.size()) ? gs[k + 1] : n;
      for (int64_t t = gs[k]; t < t1; ++t) {
        param_offsets.push_back(o);
        o += param_sizes[t];
        psi += param_sizes[t];
      }
      const int64_t size = ceil_div(o - start, unit) * unit;
      if (size > 0) {
        buckets.push_back({start, size});
        bucket_real_end.push_back(o);
      }
      o = start + size;
    }
    psi_pad = o;
    B = unit;
    for (const auto& bk : buckets) B = std::max(B, bk.second);
  } else {
    for (int64_t s : param_sizes) {
      param_offsets.push_back(psi);
      psi += s;
    }
    psi_pad = ceil_div(psi, unit) * unit;
    B = std::max(unit, (opt.bucket_elems / unit) * unit);
    for (int64_t s = 0; s < psi_pad; s += B) {
      buckets.push_back({s, std::min(B, psi_pad - s)});
      bucket_real_end.push_back(std::min(psi, s + std::min(B, psi_pad - s)));
    }
  }
  p_numel = psi_pad / divl(P);
  g_numel = (G == LV_N) ? 0 : psi_pad / divl(G);
  os_numel = psi_pad / divl(OS);
  if ((G != OS || G == LV_N) && N > 1) {   // reduced gradient needs its own slots
    // two-phase step: all of g_hat is reduced before the first update
    nslots = opt.two_phase ? (int)buckets.size() : opt.pipeline_depth + 1;
    ghat_slot = B / divl(OS);
  }
  const int64_t C = B / N;
  stage_i_len = B / M;       // largest intra block: a whole chunk (RS_I)
  stage_e_len = C;
  p1_len = B / M;
  sown_len = C;
  land_len = int64_t(M - 1) * (B / M) + int64_t(g - 1) * C;
  buf_len[BUF_GRAD] = opt.grad_slots > 0 ? std::min<int64_t>(psi_pad, int64_t(opt.grad_slots) * B) : psi_pad;
  buf_len[BUF_PARAM] = p_numel;
  buf_len[BUF_GSHARD] = g_numel;
  buf_len[BUF_GHAT] = int64_t(nslots) * ghat_slot;
  buf_len[BUF_STAGE_I] = (N > 1) ? 2 * kStageSets * stage_i_len : 0;
  buf_len[BUF_STAGE_E] = (N > 1) ? 2 * kStageSets * stage_e_len : 0;
  buf_len[BUF_P1] = (N > 1) ? kStageSets * p1_len : 0;
  buf_len[BUF_SOWN] = (N > 1) ? kStageSets * sown_len : 0;
  buf_len[BUF_LAND] = (N > 1 && ((opt.topology == 3 && opt.push) || (opt.ce_reduce && G == LV_I)))
                          ? kStageSets * land_len : 0;
  buf_len[BUF_GACC] = (opt.accum && G == LV_N) ? psi_pad : 0;
  buf_len[BUF_WIN] = (opt.windows > 0 && P != LV_N && N > 1) ? int64_t(opt.windows) * B : 0;
  buf_len[BUF_XW] = (opt.wire == 4 && opt.topology == 4 && N > 1) ? B : 0;
  acc_kind = !opt.accum ? -1 : (G == LV_N ? BUF_GACC : BUF_GSHARD);
  if (opt.params_only) {   // frozen tensors: no gradient, no optimizer state, no staging
    for (int k = 0; k < BUF_NKINDS; ++k)
      if (k != BUF_PARAM && k != BUF_WIN) buf_len[k] = 0;
    g_numel = os_numel = 0;
    acc_kind = -1;
  }
  // raw gradients and parameters are bf16; every buffer that holds a
  // reduction partial or g_hat carries the wire type
  for (int k = 0; k < BUF_NKINDS; ++k) esz[k] = opt.wire;
  esz[BUF_GRAD] = esz[BUF_PARAM] = esz[BUF_WIN] = 2;
  int64_t off = 0;
  for (int k = 0; k < BUF_NKINDS; ++k) {
    buf_off[k] = off;
    off += round_up(buf_len[k] * esz[k], 2 * kAlignElems);
  }
  region_bytes = off;
}

void Planner::build_schedule() {
  sched.assign(buckets.size(), BucketSchedule());
  int topo = opt.topology;   // per bucket: the one-shot topology hands large buckets to HO-Ring
  // primitive names (reporting; mirrors oracle.accounting.step_ops)
  grad_ops.clear();
  rest_ops.clear();
  if (G == LV_I) {
    grad_ops = {"RS_I", OS == LV_G ? "RS_E" : "AR_E"};
  } else {
    grad_ops = {"HO_RS"};
    if (OS == LV_I) grad_ops.push_back("AG_E");
    if (OS == LV_N) grad_ops.push_back("HO_AG");
  }
  if (OS != P) rest_ops = {OS == LV_G ? (P == LV_I ? "AG_E" : "HO_AG") : "AG_I"};

  const bool push = opt.push;
  // OS = I, G = I at g = 2 (R31): the inter all-reduce of the intra partials
  // (RS_E + AG_E) runs inside the Adam kernel, which folds the
  // same-position peer's partial (pulled over NVLink) with its own.  For g = 2
  // R_2(j; S_0, S_1) = S_{j+1} (+) S_j is one bf16 add, commutative, so both
  // segments of the chunk get the ring's bits; each rank's partial is read
  // once by its peer: (g-1)/g * 2 * chunk = chunk elements, the ring's bytes.
  // G = N (NNI, INI): the same fold after an RS_I of the raw gradients into the
  // g_hat slot (HO-RS at g = 2 minus its inter part; two-step and direct give the
  // same bits); the slot is reused pipeline_depth + 1 buckets later, so that
  // RS_I's round-0 barrier also waits for the inter peer (whose Adam read it).
  // M = 1 (groups of one GPU, I == N): the partials are the raw gradients
  // themselves (scaled by 1/N on read), so Adam folds the peer's raw bucket
  // with its own for every OS != G code: the whole all-reduce in the update.
  const bool topo_ok = opt.topology == 0 || opt.topology == 1 || opt.topology == 3 || opt.topology == 6;
  const bool fuse_ar_e = opt.fuse_ar_e && !push && N > 1 && g == 2 &&
                         ((M > 1 && OS == LV_I && (G == LV_I ? opt.topology != 4 : topo_ok)) ||
                          (M == 1 && OS != LV_G && topo_ok));
  fused_allreduce = fuse_ar_e;
  for (size_t b = 0; b < buckets.size(); ++b) {
    BucketSchedule& S = sched[b];
    const int64_t s = buckets[b].first, n = buckets[b].second;
    // one-shot collectives win up to 256 MiB buckets at 2x2 (2 barriers instead
    // of 4, rotated peer order: 666 vs 682 us at 256 MiB; 512 MiB buckets 2604 vs
    // 2573 us, profiles/r02/oneshot_a2a_rotated_4gpu.jsonl), so larger buckets
    // run the HO-Ring schedules (the same canonical bits)
    topo = (opt.topology == 6 && n * opt.wire > oneshot_max_bytes()) ? 0 : opt.topology;
    const int64_t C = n / N, chunk = n / M;
    const int par = int(b % kStageSets);
    S.reduce.n_ranks = S.gather.n_ranks = S.accum.n_ranks = S.reduce_acc.n_ranks = S.window.n_ranks = N;
    S.nccl_reduce.assign(N, {});
    S.nccl_gather.assign(N, {});

    int src_kind = BUF_GRAD;   // BUF_GACC while emitting the G = N post-accumulation reduction
    // raw gradients: the flat buffer, or bucket slot b % K of a streamed step
    const int64_t gbase = opt.grad_slots > 0 ? int64_t(b % opt.grad_slots) * B : s;
    auto grad = [&](int r, int64_t o) { return Ref{r, src_kind, (src_kind == BUF_GRAD ? gbase : s) + o}; };
    auto gshard = [&](int r, int64_t o) { return Ref{r, BUF_GSHARD, s / divl(G) + o}; };
    auto ghat_base = [&](int r) {
      if (G == OS && G != LV_N) return Ref{r, BUF_GSHARD, s / divl(G)};
      return Ref{r, BUF_GHAT, int64_t(b % nslots) * ghat_slot};
    };
    auto param_base = [&](int r) { return Ref{r, BUF_PARAM, s / divl(P)}; };
    auto stage_i = [&](int r, int slot) { return Ref{r, BUF_STAGE_I, int64_t(par * 2 + slot) * stage_i_len}; };
    auto stage_e = [&](int r, int slot) { return Ref{r, BUF_STAGE_E, int64_t(par * 2 + slot) * stage_e_len}; };
    (void)stage_e;
    auto p1 = [&](int r) { return Ref{r, BUF_P1, int64_t(par) * p1_len}; };
    auto sown = [&](int r) { return Ref{r, BUF_SOWN, int64_t(par) * sown_len}; };
    // where the reduced segment of rank r lands (OS-residency layout of g_hat)
    auto dest_seg = [&](int r) {
      const int j = grp(r), p = pos(r);
      if (OS == LV_G) return ghat_base(r);
      if (OS == LV_I) return at(ghat_base(r), int64_t(j) * C);
      return at(ghat_base(r), int64_t(seg(j, p)) * C);
    };
    auto group_ranks = [&](int j) {
      std::vector<int> v;
      for (int p = 0; p < M; ++p) v.push_back(rank_of(j, p));
      return v;
    };
    auto pos_ranks = [&](int p) {
      std::vector<int> v;
      for (int j = 0; j < g; ++j) v.push_back(rank_of(j, p));
      return v;
    };
    auto one = [](int64_t off, int64_t len) { return std::vector<Piece>{{off, len, 0}}; };

    auto land_i = [&](int r, int slot) {
      return Ref{r, BUF_LAND, int64_t(par) * land_len + int64_t(slot) * chunk};
    };
    auto land_e = [&](int r, int slot) {
      return Ref{r, BUF_LAND, int64_t(par) * land_len + int64_t(M - 1) * chunk + int64_t(slot) * C};
    };
    // foreign-group segments of chunk c for group j: 1 or 2 contiguous pieces
    auto foreign_pieces = [&](int j, int c) {
      std::vector<Piece> v;
      const int64_t base = int64_t(c) * g * C;
      if (j > 0) v.push_back({base, int64_t(j) * C, 0});
      if (j < g - 1) v.push_back({base + int64_t(j + 1) * C, int64_t(g - 1 - j) * C, int64_t(j) * C});
      return v;
    };

    // ---- world-reaching RS producing g_hat segments at dest_seg (G in {N, G}).
    // Returns rounds used.
    // one-shot (NVSwitch, pull): rank r folds segment k of every rank's raw
    // gradients in one round, in the segment owner's canonical order (R2):
    // blocks j' = owner-group + 1 .. owner-group, inside each the positions
    // owner-position + 1 .. owner-position (a nested fold when g > 1 and M > 1)
    auto oneshot_task = [&](int k, Ref dst) {
      Task t;
      t.n = C;
      const int jo = k % g, po = k / g;   // segment k = p * g + j (R1)
      for (int bj = 1; bj <= g; ++bj)
        for (int bp = 1; bp <= M; ++bp) t.in[t.nin++] = grad(rank_of((jo + bj) % g, (po + bp) % M), int64_t(k) * C);
      if (g > 1 && M > 1) {
        t.nest = M;
        t.nblk = g;
      }
      t.dst = dst;
      return t;
    };
    auto emit_world_rs = [&](Launch& L, int round0) -> int {
      if (topo == 6) {
        for (int r = 0; r < N; ++r) L.add(round0, r, oneshot_task(seg(grp(r), pos(r)), dest_seg(r)));
        return 1;
      }
      if (topo == 0) {  // HO-Ring RS (R16/R17)
        int R1 = 0;
        if (g > 1 && M > 1) {   // phase 1: intra ring RS of the foreign-group segments
          for (int j = 0; j < g; ++j) {
            auto gr = group_ranks(j);
            R1 = ring_rs(L, push, gr, [&, j](int c) { return foreign_pieces(j, c); },
                         [&, gr](int q, int, const Piece& pc) { return grad(gr[q], pc.src_off); },
                         [&, gr](int q, int slot) { return stage_i(gr[q], slot); },
                         [&, gr](int q) { return p1(gr[q]); }, round0);
          }
        }
        // phase 2: inter ring (i) concurrent with the intra own-segment ring (ii)
        std::vector<FinalIn> intra_fin(N), inter_fin(N);
        int off_i = 0, off_e = 0;
        if (M > 1) {
          for (int j = 0; j < g; ++j) {
            auto gr = group_ranks(j);
            auto rb = ring_rs_body(L, push, gr, [&, j](int c) { return one(int64_t(seg(j, c)) * C, C); },
                                   [&, gr](int q, int, const Piece& pc) { return grad(gr[q], pc.src_off); },
                                   [&, gr](int q, int slot) { return stage_i(gr[q], slot); }, round0 + R1);
            off_i = rb.final_off;
            for (int q = 0; q < M; ++q) intra_fin[gr[q]] = rb.fin[q];
          }
        }
        if (g > 1) {
          for (int p = 0; p < M; ++p) {
            auto pr = pos_ranks(p);
            auto contrib = [&, pr, p](int q, int c, const Piece&) {
              if (M > 1 && c != q) return at(p1(pr[q]), int64_t(c < q ? c : c - 1) * C);
              return grad(pr[q], int64_t(seg(c, p)) * C);   // M == 1, or the own segment
            };
            auto rb = ring_rs_body(L, push, pr, [&](int) { return one(0, C); }, contrib,
                                   [&, pr](int q, int slot) { return stage_e(pr[q], slot); }, round0 + R1);
            off_e = rb.final_off;
            for (int q = 0; q < g; ++q) inter_fin[pr[q]] = rb.fin[q];
          }
        }
        const int rf = round0 + R1 + std::max(off_i, off_e);
        for (int r = 0; r < N; ++r) {
          Ref d = dest_seg(r);
          if (g == 1) {
            L.add(rf, r, make_task(C, {intra_fin[r].pin[0], intra_fin[r].own[0]}, d));
          } else if (M == 1) {
            L.add(rf, r, make_task(C, {inter_fin[r].pin[0], inter_fin[r].own[0]}, d));
          } else if (round0 + R1 + off_i == rf) {   // fused: ((intra_in (+) x_own) (+) inter_in)
            L.add(rf, r, make_task(C, {intra_fin[r].pin[0], intra_fin[r].own[0], inter_fin[r].pin[0]}, d));
          } else {   // intra ring finished earlier: stash S_j, combine it last
            L.add(round0 + R1 + off_i, r, make_task(C, {intra_fin[r].pin[0], intra_fin[r].own[0]}, sown(r)));
            L.add(rf, r, make_task(C, {inter_fin[r].pin[0], sown(r)}, d));
          }
        }
        return rf - round0 + 1;
      }
      if (topo == 1 || topo == 5) {  // two-step: RS_I into P1, then RS_E; H-Ring plans reduce this way
        int r1 = 0;
        for (int j = 0; j < g; ++j) {
          auto gr = group_ranks(j);
          r1 = ring_rs(L, push, gr, [&](int c) { return one(int64_t(c) * chunk, chunk); },
                       [&, gr](int q, int, const Piece& pc) { return grad(gr[q], pc.src_off); },
                       [&, gr](int q, int slot) { return stage_i(gr[q], slot); },
                       [&, gr](int q) { return p1(gr[q]); }, round0);
        }
        int r2 = 0;
        for (int p = 0; p < M; ++p) {
          auto pr = pos_ranks(p);
          r2 = ring_rs(L, push, pr, [&](int c) { return one(int64_t(c) * C, C); },
                       [&, pr](int q, int, const Piece& pc) { return at(p1(pr[q]), pc.src_off); },
                       [&, pr](int q, int slot) { return stage_e(pr[q], slot); },
                       [&, pr](int q) { return dest_seg(pr[q]); }, round0 + r1);
        }
        return r1 + r2;
      }
      if (topo == 2) {  // flat ring over all ranks
        std::vector<int> all;
        for (int r = 0; r < N; ++r) all.push_back(r);
        return ring_rs(L, push, all, [&](int c) { return one(int64_t(seg(grp(c), pos(c))) * C, C); },
                       [&](int q, int, const Piece& pc) { return grad(q, pc.src_off); },
                       [&](int q, int slot) { return stage_i(q, slot); }, [&](int q) { return dest_seg(q); },
                       round0);
      }
      // topo == 3: direct hierarchical (NVSwitch all-to-all): same canonical order.
      // Intra: S_j[chunk p] = R_M(p; x_(j,p+1), ..., x_(j,p)); inter: R_g(j; S_(j+1), ..., S_j).
      int rr = round0;
      if (M > 1) {
        const int64_t n1 = (g == 1) ? C : chunk;
        if (!push) {
          for (int r = 0; r < N; ++r) {
            const int j = grp(r), p = pos(r);
            Task t;
            t.n = n1;
            t.nin = M;
            for (int i = 0; i < M; ++i) t.in[i] = grad(rank_of(j, (p + 1 + i) % M), int64_t(p) * chunk);
            t.dst = (g == 1) ? dest_seg(r) : p1(r);
            L.add(rr, r, t);
          }
          rr += 1;
        } else {
          for (int r = 0; r < N; ++r) {     // every rank stores its chunk-p share into owner p's landing slot
            const int j = grp(r), pp = pos(r);
            for (int p = 0; p < M; ++p) {
              if (p == pp) continue;
              const int slot = ((pp - p - 1) % M + M) % M;
              L.add(rr, r, make_task(n1, {grad(r, int64_t(p) * chunk)}, land_i(rank_of(j, p), slot)));
            }
          }
          for (int r = 0; r < N; ++r) {     // owner folds the landed shares in canonical order
            const int p = pos(r);
            Task t;
            t.n = n1;
            t.nin = M;
            for (int i = 0; i < M - 1; ++i) t.in[i] = land_i(r, i);
            t.in[M - 1] = grad(r, int64_t(p) * chunk);
            t.dst = (g == 1) ? dest_seg(r) : p1(r);
            L.add(rr + 1, r, t);
          }
          rr += 2;
        }
      }
      if (g > 1) {
        auto spart = [&](int r, int jj) {   // group partial of segment (jj, p) held by r = (j, p)
          return (M > 1) ? at(p1(r), int64_t(jj) * C) : grad(r, int64_t(seg(jj, pos(r))) * C);
        };
        if (!push) {
          for (int r = 0; r < N; ++r) {
            const int j = grp(r), p = pos(r);
            Task t;
            t.n = C;
            t.nin = g;
            for (int i = 0; i < g; ++i) t.in[i] = spart(rank_of((j + 1 + i) % g, p), j);
            t.dst = dest_seg(r);
            L.add(rr, r, t);
          }
          rr += 1;
        } else {
          for (int r = 0; r < N; ++r) {
            const int j = grp(r), p = pos(r);
            for (int jo = 0; jo < g; ++jo) {
              if (jo == j) continue;
              const int slot = ((j - jo - 1) % g + g) % g;
              L.add(rr, r, make_task(C, {spart(r, jo)}, land_e(rank_of(jo, p), slot)));
            }
          }
          for (int r = 0; r < N; ++r) {
            const int j = grp(r);
            Task t;
            t.n = C;
            t.nin = g;
            for (int i = 0; i < g - 1; ++i) t.in[i] = land_e(r, i);
            t.in[g - 1] = spart(r, j);
            t.dst = dest_seg(r);
            L.add(rr + 1, r, t);
          }
          rr += 2;
        }
      }
      return rr - round0;
    };

    // ---- world-reaching AG of segments in place in a bucket-layout buffer.  Returns rounds used.
    auto emit_world_ag = [&](Launch& L, const std::function<Ref(int)>& base, int round0) -> int {
      if (topo == 6) {  // one-shot: every segment copied from its owner in one round
        // peers in rotated order (r+1, r+2, ...): tiles are dealt in task order, so
        // at any moment every rank reads from a different peer (no egress hotspot;
        // ascending order measured 1.8x slower at 2x2, profiles/r02/a2a_4gpu.jsonl)
        for (int r = 0; r < N; ++r)
          for (int i = 1; i < N; ++i) {
            const int x = (r + i) % N;
            const int64_t o = int64_t(seg(grp(x), pos(x))) * C;
            L.add(round0, r, make_task(C, {at(base(x), o)}, at(base(r), o)));
          }
        return 1;
      }
      if (topo == 0) {  // HO-Ring AG
        for (int j = 0; j < g; ++j) {
          auto gr = group_ranks(j);
          ring_ag(L, push, gr, [&, j](int c) { return one(int64_t(seg(j, c)) * C, C); },
                  [&, gr](int q) { return base(gr[q]); }, round0);
        }
        for (int p = 0; p < M; ++p) {
          auto pr = pos_ranks(p);
          ring_ag(L, push, pr, [&, p](int c) { return one(int64_t(seg(c, p)) * C, C); },
                  [&, pr](int q) { return base(pr[q]); }, round0);
        }
        const int ra = std::max(M - 1, g - 1);
        if (g > 1 && M > 1) {
          for (int j = 0; j < g; ++j) {
            auto gr = group_ranks(j);
            ring_ag(L, push, gr, [&, j](int c) { auto v = foreign_pieces(j, c); for (auto& pc : v) pc.blk_off = 0; return v; },
                    [&, gr](int q) { return base(gr[q]); }, round0 + ra);
          }
          return ra + M - 1;
        }
        return ra;
      }
      if (topo == 1) {  // AG_E then AG_I
        for (int p = 0; p < M; ++p) {
          auto pr = pos_ranks(p);
          ring_ag(L, push, pr, [&, p](int c) { return one(int64_t(seg(c, p)) * C, C); },
                  [&, pr](int q) { return base(pr[q]); }, round0);
        }
        for (int j = 0; j < g; ++j) {
          auto gr = group_ranks(j);
          ring_ag(L, push, gr, [&](int c) { return one(int64_t(c) * chunk, chunk); },
                  [&, gr](int q) { return base(gr[q]); }, round0 + (g - 1));
        }
        return (g - 1) + (M - 1);
      }
      if (topo == 2) {
        std::vector<int> all;
        for (int r = 0; r < N; ++r) all.push_back(r);
        return ring_ag(L, push, all, [&](int c) { return one(int64_t(seg(grp(c), pos(c))) * C, C); }, base,
                       round0);
      }
      if (topo == 5) {  // H-Ring AG: one leader (position 0) per group
        for (int j = 0; j < g; ++j) {   // phase 1: intra ring AG of the own segments
          auto gr = group_ranks(j);
          ring_ag(L, push, gr, [&, j](int c) { return one(int64_t(seg(j, c)) * C, C); },
                  [&, gr](int q) { return base(gr[q]); }, round0);
        }
        int rr = round0 + (M - 1);
        if (g > 1) {
          std::vector<int> leaders;
          for (int j = 0; j < g; ++j) leaders.push_back(rank_of(j, 0));
          // phase 2: leaders' inter ring AG of whole group blocks (M strided segments each)
          ring_ag(L, push, leaders,
                  [&](int c) {
                    std::vector<Piece> v;
                    for (int p = 0; p < M; ++p) v.push_back({int64_t(seg(c, p)) * C, C, 0});
                    return v;
                  },
                  [&](int q) { return base(leaders[q]); }, rr);
          rr += g - 1;
          // phase 3: chain broadcast of the foreign-group blocks down the positions
          for (int t = 0; t + 1 < M; ++t) {
            for (int j = 0; j < g; ++j) {
              const int src = rank_of(j, t), dst = rank_of(j, t + 1);
              for (int x = 0; x < g; ++x) {
                if (x == j) continue;
                for (int p = 0; p < M; ++p) {
                  const int64_t o = int64_t(seg(x, p)) * C;
                  if (!push) L.add(rr + t, dst, make_task(C, {at(base(src), o)}, at(base(dst), o)));
                  else L.add(rr + t, src, make_task(C, {at(base(src), o)}, at(base(dst), o)));
                }
              }
            }
          }
          rr += M - 1;
        }
        return rr - round0;
      }
      // direct: inter segments, then intra chunks
      int rr = round0;
      if (g > 1) {
        for (int r = 0; r < N; ++r) {
          const int j = grp(r), p = pos(r);
          for (int x = 0; x < g; ++x) {
            if (x == j) continue;
            if (!push) {
              const int64_t o = int64_t(seg(x, p)) * C;
              L.add(rr, r, make_task(C, {at(base(rank_of(x, p)), o)}, at(base(r), o)));
            } else {
              const int64_t o = int64_t(seg(j, p)) * C;
              L.add(rr, r, make_task(C, {at(base(r), o)}, at(base(rank_of(x, p)), o)));
            }
          }
        }
        ++rr;
      }
      if (M > 1) {
        for (int r = 0; r < N; ++r) {
          const int j = grp(r), p = pos(r);
          for (int c = 0; c < M; ++c) {
            if (c == p) continue;
            if (!push) {
              const int64_t o = int64_t(c) * chunk;
              L.add(rr, r, make_task(chunk, {at(base(rank_of(j, c)), o)}, at(base(r), o)));
            } else {
              const int64_t o = int64_t(p) * chunk;
              L.add(rr, r, make_task(chunk, {at(base(r), o)}, at(base(rank_of(j, c)), o)));
            }
          }
        }
        ++rr;
      }
      return rr - round0;
    };
    // AG_E in place in a chunk-layout buffer (segment j of chunk p at j*C)
    auto emit_ag_e = [&](Launch& L, const std::function<Ref(int)>& base, int round0) -> int {
      if (topo == 6 && g > 1) {   // one-shot: the g-1 same-position peers' segments in one round (rotated)
        for (int r = 0; r < N; ++r)
          for (int i = 1; i < g; ++i) {
            const int jj = (grp(r) + i) % g;
            const int x = rank_of(jj, pos(r));
            L.add(round0, r, make_task(C, {at(base(x), int64_t(jj) * C)}, at(base(r), int64_t(jj) * C)));
          }
        return 1;
      }
      int used = 0;
      for (int p = 0; p < M; ++p) {
        auto pr = pos_ranks(p);
        used = ring_ag(L, push, pr, [&](int c) { return one(int64_t(c) * C, C); },
                       [&, pr](int q) { return base(pr[q]); }, round0);
      }
      return used;
    };
    auto emit_ag_i = [&](Launch& L, const std::function<Ref(int)>& base, int round0) -> int {
      if (topo == 6 && M > 1) {   // one-shot: the M-1 group peers' chunks in one round (rotated)
        for (int r = 0; r < N; ++r)
          for (int i = 1; i < M; ++i) {
            const int pp = (pos(r) + i) % M;
            const int x = rank_of(grp(r), pp);
            L.add(round0, r, make_task(chunk, {at(base(x), int64_t(pp) * chunk)}, at(base(r), int64_t(pp) * chunk)));
          }
        return 1;
      }
      int used = 0;
      for (int j = 0; j < g; ++j) {
        auto gr = group_ranks(j);
        used = ring_ag(L, push, gr, [&](int c) { return one(int64_t(c) * chunk, chunk); },
                       [&, gr](int q) { return base(gr[q]); }, round0);
      }
      return used;
    };

    // RS_I of the gradients into the G residency.  Returns rounds used.
    // Copy-engine variant (opt.ce_reduce, pull): the M-1 group peers' raw chunks
    // are copied into landing slots (`pre`, run by the copy engines: raw
    // gradients do not change during a step, so no round barrier is needed),
    // then one local fold in the canonical order R_M(p; y_{p+1}, ..., y_p).
    auto emit_rs_i = [&](Launch& L, int round0, Launch* pre = nullptr,
                         std::function<Ref(int)> out = nullptr) -> int {
      if (!out) out = [&](int r) { return gshard(r, 0); };
      if (pre && opt.ce_reduce && M > 1) {
        pre->n_ranks = N;
        for (int r = 0; r < N; ++r) {
          const int j = grp(r), p = pos(r);
          Task t;
          t.n = chunk;
          t.nin = M;
          for (int i = 0; i < M - 1; ++i) {
            Ref land = land_i(r, i);
            land.raw = true;
            pre->add(0, r, make_task(chunk, {grad(rank_of(j, (p + 1 + i) % M), int64_t(p) * chunk)}, land));
            t.in[i] = land;
          }
          t.in[M - 1] = grad(r, int64_t(p) * chunk);
          t.dst = out(r);
          L.add(round0, r, t);
        }
        return 1;
      }
      if (topo == 6 && M > 1) {   // one-shot RS_I: the chunk of every group member, R_M(p; .) order
        for (int r = 0; r < N; ++r) {
          const int j = grp(r), p = pos(r);
          Task t;
          t.n = chunk;
          for (int i = 1; i <= M; ++i) t.in[t.nin++] = grad(rank_of(j, (p + i) % M), int64_t(p) * chunk);
          t.dst = out(r);
          L.add(round0, r, t);
        }
        return 1;
      }
      int r1 = 0;
      for (int j = 0; j < g; ++j) {
        auto gr = group_ranks(j);
        r1 = ring_rs(L, push, gr, [&](int c) { return one(int64_t(c) * chunk, chunk); },
                     [&, gr](int q, int, const Piece& pc) { return grad(gr[q], pc.src_off); },
                     [&, gr](int q, int slot) { return stage_i(gr[q], slot); },
                     [&, gr, out](int q) { return out(gr[q]); }, round0);
      }
      return r1;
    };
    // RS_E from the G residency; in place + AG_E for OS = I (all-reduce)
    auto emit_rs_e = [&](Launch& L, int round0) {
      if (topo == 6 && g > 1) {   // one-shot RS_E: segment j of the g same-position partials, R_g(j; .) order
        for (int r = 0; r < N; ++r) {
          const int j = grp(r), p = pos(r);
          Task t;
          t.n = C;
          for (int i = 1; i <= g; ++i) t.in[t.nin++] = gshard(rank_of((j + i) % g, p), int64_t(j) * C);
          t.dst = dest_seg(r);
          L.add(round0, r, t);
        }
        if (OS == LV_I) emit_ag_e(L, [&](int r) { return ghat_base(r); }, round0 + 1);
        return;
      }
      int r2 = 0;
      for (int p = 0; p < M; ++p) {
        auto pr = pos_ranks(p);
        r2 = ring_rs(L, push, pr, [&](int c) { return one(int64_t(c) * C, C); },
                     [&, pr](int q, int, const Piece& pc) { return gshard(pr[q], pc.src_off); },
                     [&, pr](int q, int slot) { return stage_e(pr[q], slot); },
                     [&, pr](int q) { return dest_seg(pr[q]); }, round0);
      }
      if (OS == LV_I) emit_ag_e(L, [&](int r) { return ghat_base(r); }, round0 + r2);
    };
    // G in {N, G}: world RS (+ AG_E / world AG of g_hat for OS = I / N)
    auto emit_world_reduce = [&](Launch& L) {
      // one-shot all-reduce: every rank folds every segment in one round, reading
      // (N-1) B instead of the 2(N-1)/N B of one-shot RS + AG (two rounds); worth
      // it while the extra bytes cost less than a barrier (~10 us ~ 6 MB of
      // NVLink): always at N = 2 (equal bytes), small buckets otherwise
      const int64_t extra = (int64_t)(N - 1) * (N - 2) * n * opt.wire / N;
      if (topo == 6 && OS == LV_N && (N == 2 || extra <= kOneRoundExtraBytes)) {
        for (int r = 0; r < N; ++r)
          for (int i = 0; i < N; ++i) {   // segments in rotated order, like the one-shot AG
            const int k = (seg(grp(r), pos(r)) + i) % N;
            L.add(0, r, oneshot_task(k, at(ghat_base(r), int64_t(k) * C)));
          }
        return;
      }
      int used = emit_world_rs(L, 0);
      if (OS == LV_I) emit_ag_e(L, [&](int r) { return ghat_base(r); }, used);
      if (OS == LV_N) emit_world_ag(L, [&](int r) { return ghat_base(r); }, used);
    };

    if (N > 1 && topo != 4) {
      Launch& L = S.reduce;
      if (fuse_ar_e && M == 1) {
        // nothing to reduce inside a group of one
      } else if (G == LV_I) {
        const int r1 = emit_rs_i(L, 0, &S.reduce_pre);
        if (!fuse_ar_e) emit_rs_e(L, r1);
      } else if (fuse_ar_e) {
        emit_rs_i(L, 0, nullptr, [&](int r) { return ghat_base(r); });
      } else {
        emit_world_reduce(L);
      }
      // ---- gradient accumulation (R27): per micro-batch only the
      // G-level reduction, into the accumulator; the rest once, from it
      if (opt.accum) {
        if (G == LV_G) {
          emit_world_rs(S.accum, 0);          // lands in the G residency (dest_seg)
        } else if (G == LV_I) {
          emit_rs_i(S.accum, 0, &S.accum_pre);
          if (!fuse_ar_e) emit_rs_e(S.reduce_acc, 0);   // else folded into Adam (below)
        } else {
          for (int r = 0; r < N; ++r) S.accum.add(0, r, make_task(n, {grad(r, 0)}, Ref{r, BUF_GACC, s}));
          src_kind = BUF_GACC;
          emit_world_reduce(S.reduce_acc);
          src_kind = BUF_GRAD;
        }
      }
      // ---- parameter restore
      Launch& Lg = S.gather;
      // ---- fused parameter all-gather (B200 design: the bf16 cast lands in the
      // consumers' buffers straight from the Adam kernel over NVLink).  Only
      // where the restore is ONE ring, so bytes per link class are unchanged:
      // AG_E (P = I, OS = G: the g-1 same-position ranks), AG_I (P = N, OS = I:
      // the M-1 group members), HO_AG with M = 1 or g = 1 (all other ranks).
      const bool one_ring = (OS == LV_G && P == LV_I) || (OS == LV_I && P == LV_N) ||
                            (OS == LV_G && P == LV_N && (M == 1 || g == 1));
      const int n_cons = (OS == LV_G && P == LV_I) ? g - 1 : ((OS == LV_I) ? M - 1 : N - 1);
      if (opt.fuse_gather > 0 && one_ring && n_cons <= kMaxPush && n_cons > 0) {
        S.param_push.assign(N, {});
        for (int r = 0; r < N; ++r) {
          const int j = grp(r), p = pos(r);
          Ref mine = param_base(r);
          if (P == LV_I) mine = at(mine, int64_t(j) * C);
          else if (OS == LV_G) mine = at(mine, int64_t(seg(j, p)) * C);
          else mine = at(mine, int64_t(p) * chunk);
          for (int x = 0; x < N; ++x) {
            if (x == r) continue;
            const bool cons = (OS == LV_G && P == LV_I) ? (pos(x) == p) : (OS == LV_I ? grp(x) == j : true);
            if (cons) S.param_push[r].push_back(Ref{x, BUF_PARAM, mine.off});
          }
        }
      }
      // ---- forward/backward parameter all-gather into a window (P = I / G):
      // round 0 copies the own P shard into its place, then the ring AG in place
      // (P = I: AG_I, "intra-group all-gather"; P = G: the world AG)
      if (opt.windows > 0 && P != LV_N) {
        auto win = [&](int r) { return Ref{r, BUF_WIN, 0}; };
        for (int r = 0; r < N; ++r) {
          int64_t b0, e0;
          residency(P, r, (int64_t)b, &b0, &e0);
          S.window.add(0, r, make_task(e0 - b0, {param_base(r)}, at(win(r), b0 - s)));
        }
        if (P == LV_I) emit_ag_i(S.window, win, 1);
        else emit_world_ag(S.window, win, 1);
        S.window.final_barrier = true;   // peers are done reading the slot before it is reused
      }
      if (S.param_push.empty()) {
        if (OS == LV_G && P == LV_I) emit_ag_e(Lg, param_base, 0);
        if (OS == LV_G && P == LV_N) emit_world_ag(Lg, param_base, 0);
        if (OS == LV_I && P == LV_N) emit_ag_i(Lg, param_base, 0);
      }
      // drop rounds that ended up empty for every rank (degenerate splits)
      auto finish = [&](Launch* Lp) {
        const bool is_red = (Lp == &S.reduce || Lp == &S.reduce_acc);
        std::vector<std::vector<Ref>>& gin = (Lp == &S.reduce_acc) ? S.ghat_in_acc : S.ghat_in;
        std::vector<std::vector<std::vector<Task>>> kept;
        for (auto& rnd : Lp->rounds) {
          bool any = false;
          for (auto& v : rnd) any = any || !v.empty();
          if (any) kept.push_back(rnd);
        }
        Lp->rounds.swap(kept);
        // OS = G: the last fold of the reduction (the owner's final hop) moves
        // into the Adam kernel, which reads its inputs directly (push: all
        // local; pull: the predecessor's partial over NVLink): g_hat is never
        // written to / re-read from HBM.  The launch then ends with a barrier
        // that also covers the ranks the fused Adam reads (final_extra).
        if (is_red && OS == LV_G && opt.fuse_final && !Lp->rounds.empty()) {
          gin.assign(N, {});
          Lp->final_extra.assign(N, 0);
          auto& last = Lp->rounds.back();
          for (int r = 0; r < N; ++r) {
            const Ref d = dest_seg(r);
            for (size_t i = 0; i < last[r].size(); ++i) {
              const Task& t = last[r][i];
              if (t.dst.rank == d.rank && t.dst.kind == d.kind && t.dst.off == d.off && t.n == C &&
                  t.nin <= kMaxAdamIn && t.nest <= 1) {
                for (int k = 0; k < t.nin; ++k) gin[r].push_back(t.in[k]);
                last[r].erase(last[r].begin() + i);
                break;
              }
            }
          }
          for (int r = 0; r < N; ++r)
            for (const Ref& x : gin[r])
              if (x.rank != r) {
                Lp->final_extra[r] |= uint64_t(1) << x.rank;
                Lp->final_extra[x.rank] |= uint64_t(1) << r;
              }
          bool any = false;
          for (auto& v : last) any = any || !v.empty();
          if (!any) Lp->rounds.pop_back();
          Lp->final_barrier = true;
        }
        // a launch whose last round stores into peers ends with a barrier so the
        // data has landed before the peer's next kernel reads it
        if (!Lp->rounds.empty()) {
          for (int r = 0; r < N; ++r)
            for (const Task& t : Lp->rounds.back()[r])
              if (t.dst.rank != r) Lp->final_barrier = true;
        }
        if (Lp->final_extra.empty()) Lp->final_extra.assign(N, 0);
      };
      for (Launch* Lp : {&S.reduce, &S.gather, &S.accum, &S.reduce_acc, &S.window}) finish(Lp);
      if (fuse_ar_e) {
        // Adam reads [peer partial, own partial] over the whole chunk; the RS_I
        // launch ends with a barrier that covers the inter peer it reads
        auto part = [&](int r) { return M == 1 ? grad(r, 0) : (G == LV_I ? gshard(r, 0) : ghat_base(r)); };
        const bool slot_reuse = M > 1 && G == LV_N;
        S.ghat_in.assign(N, {});
        S.reduce.final_extra.assign(N, 0);
        if (slot_reuse) S.reduce.first_extra.assign(N, 0);
        for (int r = 0; r < N; ++r) {
          const int y = rank_of(1 - grp(r), pos(r));
          S.ghat_in[r] = {part(y), part(r)};
          S.reduce.final_extra[r] |= uint64_t(1) << y;
          if (slot_reuse) S.reduce.first_extra[r] |= uint64_t(1) << y;
        }
        S.reduce.final_barrier = true;
        // gradient accumulation, G = I: the accumulated intra partials sit in the
        // G residency; the step after the last micro-batch folds them in Adam too
        // (no barrier launch: paro_accumulate ends with an all-peer barrier, which
        // already orders every peer's accumulator writes before this step, and the
        // step-end barrier orders Adam's peer reads before the next accumulation)
        if (opt.accum && G == LV_I) {
          S.ghat_in_acc.assign(N, {});
          S.reduce_acc.final_extra.assign(N, 0);
          for (int r = 0; r < N; ++r) {
            const int y = rank_of(1 - grp(r), pos(r));
            S.ghat_in_acc[r] = {gshard(y, 0), gshard(r, 0)};
          }
          S.reduce_acc.final_barrier = false;
        }
      }
      // fused gather, auto mode: only when no collective rounds run beside Adam
      // (the whole reduction fused too); beside a rounds kernel the separate
      // all-gather launch measured faster (profiles/r01/sweep_fuse_gather_2x2*.jsonl)
      if (opt.fuse_gather == 1 && !S.param_push.empty() && !S.reduce.rounds.empty()) {
        S.param_push.clear();
        if (OS == LV_G && P == LV_I) emit_ag_e(Lg, param_base, 0);
        if (OS == LV_G && P == LV_N) emit_world_ag(Lg, param_base, 0);
        if (OS == LV_I && P == LV_N) emit_ag_i(Lg, param_base, 0);
        finish(&Lg);
      }
    } else if (N == 1 && opt.accum) {   // one rank: the accumulation is a local fold
      S.accum.add(0, 0, make_task(n, {grad(0, 0)}, Ref{0, acc_kind, s}));
      S.accum.final_extra.assign(1, 0);
      S.reduce_acc.final_extra.assign(1, 0);
      S.reduce.final_extra.assign(1, 0);
      S.gather.final_extra.assign(1, 0);
    } else if (N > 1 && topo == 4) {  // NCCL comparator
      // fp32 wire: the raw bf16 gradients are first pre-scaled into an fp32
      // bucket (a local round of the rounds kernel), which NCCL then reduces
      auto xsrc = [&](int r) { return opt.wire == 4 ? Ref{r, BUF_XW, 0} : grad(r, 0); };
      if (opt.wire == 4)
        for (int r = 0; r < N; ++r) S.reduce.add(0, r, make_task(n, {grad(r, 0)}, xsrc(r)));
      for (int r = 0; r < N; ++r) {
        auto& red = S.nccl_reduce[r];
        auto& gat = S.nccl_gather[r];
        const int j = grp(r);
        if (G == LV_I) {
          red.push_back({NcclCall::RS, NcclCall::INTRA, xsrc(r), gshard(r, 0), chunk});
          if (OS == LV_G) red.push_back({NcclCall::RS, NcclCall::INTER, gshard(r, 0), dest_seg(r), C});
          else red.push_back({NcclCall::AR, NcclCall::INTER, gshard(r, 0), gshard(r, 0), chunk});
        } else {
          red.push_back({NcclCall::RS, NcclCall::INTRA, xsrc(r), p1(r), chunk});
          red.push_back({NcclCall::RS, NcclCall::INTER, p1(r), dest_seg(r), C});
          if (OS == LV_I) red.push_back({NcclCall::AG, NcclCall::INTER, dest_seg(r), ghat_base(r), C});
          if (OS == LV_N) {
            Ref cb = at(ghat_base(r), int64_t(pos(r)) * chunk);
            red.push_back({NcclCall::AG, NcclCall::INTER, dest_seg(r), cb, C});
            red.push_back({NcclCall::AG, NcclCall::INTRA, cb, ghat_base(r), chunk});
          }
        }
        if (OS == LV_G && P == LV_I)
          gat.push_back({NcclCall::AG, NcclCall::INTER, at(param_base(r), int64_t(j) * C), param_base(r), C});
        if (OS == LV_G && P == LV_N) {
          Ref cb = at(param_base(r), int64_t(pos(r)) * chunk);
          gat.push_back({NcclCall::AG, NcclCall::INTER, at(cb, int64_t(j) * C), cb, C});
          gat.push_back({NcclCall::AG, NcclCall::INTRA, cb, param_base(r), chunk});
        }
        if (OS == LV_I && P == LV_N)
          gat.push_back({NcclCall::AG, NcclCall::INTRA, at(param_base(r), int64_t(pos(r)) * chunk),
                         param_base(r), chunk});
      }
    }

    // ---- Adam placement per rank
    S.os_len = n / divl(OS);
    S.ghat.resize(N);
    S.param.resize(N);
    S.os_off.resize(N);
    for (int r = 0; r < N; ++r) {
      const int j = grp(r), p = pos(r);
      S.os_off[r] = s / divl(OS);
      S.ghat[r] = (N == 1) ? grad(r, 0) : ghat_base(r);
      if (S.ghat_in.size() != (size_t)N || S.ghat_in[r].empty()) S.ghat_in.resize(N), S.ghat_in[r] = {S.ghat[r]};
      if (opt.accum && (S.ghat_in_acc.size() != (size_t)N || S.ghat_in_acc[r].empty())) {
        S.ghat_in_acc.resize(N);
        S.ghat_in_acc[r] = {(N == 1) ? Ref{r, acc_kind, s} : ghat_base(r)};   // materialised g_hat
      }
      Ref pb = param_base(r);
      if (P == OS) S.param[r] = pb;
      else if (P == LV_I) S.param[r] = at(pb, int64_t(j) * C);              // OS = G
      else if (OS == LV_G) S.param[r] = at(pb, int64_t(seg(j, p)) * C);     // P = N
      else S.param[r] = at(pb, int64_t(p) * chunk);                         // P = N, OS = I
    }
  }
}

// Every transfer must stay inside its buffer kind (caught on the CPU, before
// any kernel could fault on a bad schedule).
void Planner::validate_refs() const {
  auto ok = [&](const Ref& r, int64_t n) {
    return r.rank >= 0 && r.rank < N && r.kind >= 0 && r.kind < BUF_NKINDS && r.off >= 0 &&
           r.off + n <= buf_len[r.kind] && r.off % 8 == 0;
  };
  for (size_t b = 0; b < sched.size(); ++b) {
    const BucketSchedule& S = sched[b];
    for (const Launch* L : {&S.reduce, &S.gather, &S.accum, &S.reduce_acc, &S.window, &S.reduce_pre, &S.accum_pre})
      for (const auto& rnd : L->rounds)
        for (const auto& v : rnd)
          for (const Task& t : v) {
            if (t.n <= 0 || t.n % 8 != 0 || t.nin < 1 || t.nin > kMaxIn ||
                (L == &S.accum && t.dst.kind == acc_kind && t.nin + 1 > kMaxIn))
              throw std::logic_error("bad task shape in bucket " + std::to_string(b));
            for (int i = 0; i < t.nin; ++i)
              if (!ok(t.in[i], t.n)) throw std::logic_error("task input out of range in bucket " + std::to_string(b));
            if (!ok(t.dst, t.n)) throw std::logic_error("task output out of range in bucket " + std::to_string(b));
          }
    for (int r = 0; r < N; ++r) {
      if (!ok(S.param[r], S.os_len)) throw std::logic_error("adam output out of range in bucket " + std::to_string(b));
      for (const Ref& x : S.ghat_in[r])
        if (!ok(x, S.os_len)) throw std::logic_error("adam input out of range in bucket " + std::to_string(b));
      if (!S.param_push.empty())
        for (const Ref& x : S.param_push[r])
          if (!ok(x, S.os_len) || x.off != S.param[r].off || x.kind != BUF_PARAM)
            throw std::logic_error("fused gather target out of range in bucket " + std::to_string(b));
      for (size_t i = 0; opt.accum && i < S.ghat_in_acc[r].size(); ++i)
        if (!ok(S.ghat_in_acc[r][i], S.os_len))
          throw std::logic_error("adam input out of range in bucket " + std::to_string(b));
    }
  }
}

void Planner::count_bytes() {
  // bytes each rank sends (pull: what peers read from it; push: what it stores
  // into peers) over a list of launches plus the fused-Adam peer reads
  auto count = [&](std::initializer_list<const Launch*> Ls, const std::vector<std::vector<Ref>>* gin,
                   int64_t os_len, std::vector<int64_t>& si, std::vector<int64_t>& se,
                   const std::vector<std::vector<Ref>>* push = nullptr) {
    for (int x = 0; push && x < N && (int)push->size() == N; ++x)   // fused gather: x stores into y
      for (const Ref& y : (*push)[x]) (grp(x) == grp(y.rank) ? si[x] : se[x]) += 2 * os_len;
    for (const Launch* L : Ls)
      for (const auto& rnd : L->rounds)
        for (int x = 0; x < N; ++x)
          for (const Task& t : rnd[x]) {
            for (int i = 0; i < t.nin; ++i) {   // pull: y's bytes travel to x
              const int y = t.in[i].rank;
              if (y == x) continue;
              (grp(x) == grp(y) ? si[y] : se[y]) += esz[t.in[i].kind] * t.n;
            }
            const int z = t.dst.rank;            // push: x's bytes travel to z
            if (z != x) (grp(x) == grp(z) ? si[x] : se[x]) += esz[t.dst.kind] * t.n;
          }
    // fused final hop: the Adam kernel reads these inputs (pull: over NVLink)
    for (int x = 0; gin && x < N && (int)gin->size() == N; ++x)
      for (const Ref& y : (*gin)[x])
        if (y.rank != x) (grp(x) == grp(y.rank) ? si[y.rank] : se[y.rank]) += esz[y.kind] * os_len;
  };
  send_intra.assign(N, 0);
  send_inter.assign(N, 0);
  acc_send_intra.assign(N, 0);
  acc_send_inter.assign(N, 0);
  accstep_send_intra.assign(N, 0);
  accstep_send_inter.assign(N, 0);
  win_send_intra.assign(N, 0);
  win_send_inter.assign(N, 0);
  win_bucket_intra.assign(sched.size(), std::vector<int64_t>(N, 0));
  win_bucket_inter.assign(sched.size(), std::vector<int64_t>(N, 0));
  n_rounds = 0;
  n_comm_launches = 0;
  for (const BucketSchedule& S : sched) {
    for (const Launch* L : {&S.reduce, &S.gather}) {
      if (L->empty()) continue;
      ++n_comm_launches;
      n_rounds += (int)L->rounds.size();
    }
    count({&S.reduce_pre, &S.reduce, &S.gather}, &S.ghat_in, S.os_len, send_intra, send_inter, &S.param_push);
    {
      const size_t b = &S - sched.data();
      count({&S.window}, nullptr, 0, win_bucket_intra[b], win_bucket_inter[b]);
      for (int r = 0; r < N; ++r) {
        win_send_intra[r] += win_bucket_intra[b][r];
        win_send_inter[r] += win_bucket_inter[b][r];
      }
    }
    if (opt.accum) {
      count({&S.accum_pre, &S.accum}, nullptr, 0, acc_send_intra, acc_send_inter);
      count({&S.reduce_acc, &S.gather}, &S.ghat_in_acc, S.os_len, accstep_send_intra, accstep_send_inter,
            &S.param_push);
    }
    // NCCL comparator: ring-algorithm volumes of each call (perf only)
    for (int r = 0; r < N && opt.topology == 4; ++r) {
      for (const auto* calls : {&S.nccl_reduce[r], &S.nccl_gather[r]}) {
        for (const NcclCall& c : *calls) {
          const int k = (c.comm == NcclCall::INTRA) ? M : (c.comm == NcclCall::INTER ? g : N);
          const int64_t per = (c.kind == NcclCall::AR) ? 2 * (k - 1) * (c.count / k) : (k - 1) * c.count;
          (c.comm == NcclCall::INTRA ? send_intra[r] : send_inter[r]) += esz[c.send.kind] * per;
        }
        if (!calls->empty()) ++n_comm_launches;
      }
    }
  }
  if (opt.topology == 4) n_comm_launches /= std::max(1, N);
}

}  // namespace paro
