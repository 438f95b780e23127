// advisor.cpp — paro_advise: rank the 14 PaRO strategies for a training task
// (NEXT-4; reading R29).  Host only, no CUDA.
//
// Paper: Table 1 marks which codes are recommended for each
// training type; §3.1 trades memory (Table 2, "2Psi, 2Psi',
// 12Psi'") against communication (Table 3).  Per strategy the advisor builds
// the per-rank bytes of a mini-batch from the primitives the planner schedules
// (per-rank volumes of the ring primitives):
//   s * (per-micro-batch G-level reduction: HO-RS for G = G, RS_I for G = I)
//   + the rest of the reduction and the parameter restore, once      over Psi'
//   + 2 * s * (forward/backward parameter gather: AG_I / HO-AG)      over Psi
// and models t = intra / B_intra + inter / B_inter per rank.  For N <= 64 the
// CPU tests check these closed forms against the bytes counted from real
// plans (paro_rank_accum_send_bytes, paro_rank_gather_send_bytes).
#include <algorithm>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "paro.h"
#include "planner.h"

namespace paro {
paro_status_t api_fail(paro_status_t st, const std::string& msg);
}

namespace {

// Table 1, row by row; columns Psi' = Psi, Psi' >= Psi/6, Psi' < Psi/6, PEFT.
struct Row {
  const char* code;
  int mark[4];
};
const Row kTable1[14] = {
    {"NNN", {1, 1, 1, 1}}, {"NNI", {1, 1, 1, 1}}, {"NNG", {1, 1, 1, 0}}, {"NII", {1, 1, 1, 0}},
    {"NIG", {1, 1, 1, 0}}, {"NGG", {1, 1, 1, 0}}, {"INI", {0, 0, 0, 1}}, {"ING", {0, 1, 1, 0}},
    {"III", {0, 0, 1, 0}}, {"IIG", {1, 1, 0, 0}}, {"IGG", {1, 1, 1, 0}}, {"GNG", {0, 1, 1, 1}},
    {"GIG", {0, 1, 1, 0}}, {"GGG", {1, 1, 1, 0}},
};

enum Prim { RS_I, AG_I, RS_E, AG_E, AR_E, HO_RS, HO_AG };

// per-rank (intra, inter) elements one primitive sends on B elements
void units(Prim p, int N, int M, int64_t B, int64_t* ia, int64_t* ie) {
  const int g = N / M;
  switch (p) {
    case RS_I: case AG_I: *ia += (M - 1) * (B / M); break;
    case RS_E: case AG_E: *ie += (g - 1) * (B / N); break;
    case AR_E: *ie += 2 * (g - 1) * (B / N); break;
    case HO_RS: case HO_AG: *ia += (M - 1) * (B / M); *ie += (g - 1) * (B / N); break;
  }
}

// (per micro-batch, once) primitives of a mini-batch (R10, R27)
void minibatch_ops(const char* c, std::vector<Prim>* per_mb, std::vector<Prim>* once) {
  const char P = c[0], G = c[1], OS = c[2];
  std::vector<Prim> grad;
  if (G == 'I') grad = {RS_I, OS == 'G' ? RS_E : AR_E};
  else {
    grad = {HO_RS};
    if (OS == 'I') grad.push_back(AG_E);
    if (OS == 'N') grad.push_back(HO_AG);
  }
  std::vector<Prim> rest;
  if (OS != P) rest = {OS == 'G' ? (P == 'I' ? AG_E : HO_AG) : AG_I};
  per_mb->clear();
  once->clear();
  if (G == 'G') per_mb->push_back(HO_RS);
  else if (G == 'I') per_mb->push_back(RS_I);
  for (size_t i = (G == 'N' ? 0 : 1); i < grad.size(); ++i) once->push_back(grad[i]);
  once->insert(once->end(), rest.begin(), rest.end());
}

int64_t pad_to(int64_t x, int N) {
  const int64_t u = int64_t(N) * 64;
  return (x + u - 1) / u * u;
}

}  // namespace

extern "C" int paro_table1_column(int64_t psi, int64_t psi_trainable, int peft) {
  if (peft) return 3;
  if (psi_trainable == psi) return 0;
  return 6 * psi_trainable >= psi ? 1 : 2;
}

extern "C" paro_status_t paro_advise(const paro_advise_in_t* in, paro_advice_t* out, int cap, int* n_out) {
  if (!in || !out || !n_out) return paro::api_fail(PARO_ERR_INVALID, "null argument");
  if (cap < 14) return paro::api_fail(PARO_ERR_INVALID, "out must hold 14 entries");
  if (in->n_gpus < 1 || in->group_size < 1 || in->n_gpus % in->group_size != 0)
    return paro::api_fail(PARO_ERR_INVALID, "group_size must divide n_gpus");
  if (in->psi <= 0 || in->psi_trainable <= 0 || in->psi_trainable > in->psi)
    return paro::api_fail(PARO_ERR_INVALID, "need 0 < psi_trainable <= psi");
  if (in->accum_steps < 1) return paro::api_fail(PARO_ERR_INVALID, "accum_steps must be >= 1");
  if (!(in->bw_intra_gbs > 0.0) || !(in->bw_inter_gbs > 0.0))
    return paro::api_fail(PARO_ERR_INVALID, "bandwidths must be > 0");
  const int N = in->n_gpus, M = in->group_size;
  const int64_t s = in->accum_steps;
  const int64_t psi = pad_to(in->psi, N), pt = pad_to(in->psi_trainable, N);
  const int col = paro_table1_column(in->psi, in->psi_trainable, in->peft);
  std::vector<paro_advice_t> rows;
  try {
    for (const Row& row : kTable1) {
      const std::string err = paro::validate_strategy(row.code);
      if (!err.empty()) throw std::invalid_argument(err);
      std::vector<Prim> per_mb, once;
      minibatch_ops(row.code, &per_mb, &once);
      int64_t ia = 0, ie = 0, fa = 0, fe = 0, oa = 0, oe = 0;
      for (Prim p : per_mb) units(p, N, M, pt, &ia, &ie);
      for (Prim p : once) units(p, N, M, pt, &oa, &oe);
      if (row.code[0] != 'N') units(row.code[0] == 'I' ? AG_I : HO_AG, N, M, psi, &fa, &fe);
      paro_advice_t a;
      std::memset(&a, 0, sizeof(a));
      std::memcpy(a.code, row.code, 3);
      a.recommended = row.mark[col];
      a.intra_bytes = 2 * (s * ia + oa + 2 * s * fa);     // bf16 wire (R3)
      a.inter_bytes = 2 * (s * ie + oe + 2 * s * fe);
      a.t_comm_s = double(a.intra_bytes) / (in->bw_intra_gbs * 1e9) + double(a.inter_bytes) / (in->bw_inter_gbs * 1e9);
      auto dv = [&](char l) -> int64_t { return l == 'N' ? 1 : (l == 'I' ? M : N); };
      a.mem_bytes = 2 * psi / dv(row.code[0]) + 2 * pt / dv(row.code[1]) + 12 * pt / dv(row.code[2]);
      a.fits = double(a.mem_bytes) <= in->mem_budget_bytes ? 1 : 0;
      rows.push_back(a);
    }
  } catch (const std::exception& ex) {
    return paro::api_fail(PARO_ERR_INVALID, ex.what());
  }
  std::stable_sort(rows.begin(), rows.end(), [](const paro_advice_t& x, const paro_advice_t& y) {
    const int gx = (x.recommended && x.fits) ? 0 : 1, gy = (y.recommended && y.fits) ? 0 : 1;
    if (gx != gy) return gx < gy;
    if (x.t_comm_s != y.t_comm_s) return x.t_comm_s < y.t_comm_s;
    if (x.mem_bytes != y.mem_bytes) return x.mem_bytes < y.mem_bytes;
    return std::strcmp(x.code, y.code) < 0;
  });
  for (size_t i = 0; i < rows.size(); ++i) out[i] = rows[i];
  *n_out = (int)rows.size();
  return PARO_OK;
}
