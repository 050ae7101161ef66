// Host-side planner: parse the einsum model string, build einstr_l = swap(model, l), and
// lower each factor update to the streamed (row, col, bond) form of DESIGN.md §Planner.
//
// Paper: model family eq:contraction_structure / eq:einsum; einstr_l and swap
// (P:140-149); Algorithm 1 lines 1-3.  Everything here is host metadata.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <sstream>

#include "nef_internal.h"
#include "../../include/nef.h"

namespace nef {

namespace {

bool is_letter(char c) { return (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z'); }

int parse_model(const char* s, std::vector<std::string>& ops, std::string& out, std::string& err) {
  if (!s) { err = "null einsum string"; return NEF_E_ARG; }
  std::string t;
  for (const char* p = s; *p; ++p)
    if (*p != ' ' && *p != '\t' && *p != '\n') t.push_back(*p);
  size_t arrow = t.find("->");
  if (arrow == std::string::npos || t.find("->", arrow + 1) != std::string::npos) {
    err = "missing or repeated '->'";
    return NEF_E_PARSE;
  }
  std::string lhs = t.substr(0, arrow);
  out = t.substr(arrow + 2);
  ops.clear();
  std::string cur;
  for (size_t i = 0; i <= lhs.size(); ++i) {
    if (i == lhs.size() || lhs[i] == ',') {
      if (cur.empty()) { err = "empty operand"; return NEF_E_PARSE; }
      ops.push_back(cur);
      cur.clear();
    } else {
      cur.push_back(lhs[i]);
    }
  }
  for (auto& op : ops) {
    for (char c : op)
      if (!is_letter(c)) { err = std::string("illegal character '") + c + "' in operand " + op; return NEF_E_PARSE; }
    std::set<char> seen(op.begin(), op.end());
    if (seen.size() != op.size()) { err = "repeated index in operand " + op; return NEF_E_PARSE; }
  }
  if (out.empty()) { err = "empty output"; return NEF_E_PARSE; }
  for (char c : out)
    if (!is_letter(c)) { err = std::string("illegal character '") + c + "' in output"; return NEF_E_PARSE; }
  if (std::set<char>(out.begin(), out.end()).size() != out.size()) { err = "repeated output index"; return NEF_E_PARSE; }
  for (char c : out) {
    bool found = false;
    for (auto& op : ops) found |= op.find(c) != std::string::npos;
    if (!found) { err = std::string("output index '") + c + "' absent from operands"; return NEF_E_PARSE; }
  }
  if ((int)out.size() > kMaxModes) { err = "too many observed modes"; return NEF_E_UNSUPPORTED; }
  for (auto& op : ops)
    if ((int)op.size() > kMaxDims) { err = "operand with too many indices"; return NEF_E_UNSUPPORTED; }
  return NEF_OK;
}

bool mul_overflow(int64_t a, int64_t b, int64_t* r) { return __builtin_mul_overflow(a, b, r); }

int64_t prod_idx(const Plan& p, const std::string& idx) {
  int64_t n = 1;
  for (char c : idx) n *= p.dims[(int)c];
  return n;
}

// row-major strides of a tensor with index string `idx`
int64_t stride_of(const Plan& p, const std::string& idx, char c) {
  size_t pos = idx.find(c);
  if (pos == std::string::npos) return 0;
  int64_t s = 1;
  for (size_t k = pos + 1; k < idx.size(); ++k) s *= p.dims[(int)idx[k]];
  return s;
}

struct Operand {
  BufRef buf;
  std::string idx;
};

// bump allocator over the workspace (bytes, 256-aligned)
struct Bump {
  int64_t off = 0;
  std::vector<std::pair<int64_t, int64_t>> log;   // every region handed out: [offset, end)
  int64_t take(int64_t bytes) {
    int64_t o = (off + 255) / 256 * 256;
    off = o + std::max<int64_t>(bytes, 0);
    log.emplace_back(o, off);
    return o;
  }
};

EinStep make_step(const Plan& p, const Operand& A, const Operand* B, const std::string& cidx, BufRef c) {
  EinStep st;
  st.a = A.buf;
  st.a_idx = A.idx;
  if (B) { st.b = B->buf; st.b_idx = B->idx; }
  st.c = c;
  st.c_idx = cidx;
  st.nout = (int)cidx.size();
  for (int d = 0; d < st.nout; ++d) {
    char ch = cidx[d];
    st.odim[d] = p.dims[(int)ch];
    st.as_o[d] = stride_of(p, A.idx, ch);
    st.bs_o[d] = B ? stride_of(p, B->idx, ch) : 0;
    st.out_size *= st.odim[d];
  }
  std::string all = A.idx + (B ? B->idx : std::string());
  std::string sum;
  for (char ch : all)
    if (cidx.find(ch) == std::string::npos && sum.find(ch) == std::string::npos) sum.push_back(ch);
  st.nsum = (int)sum.size();
  for (int d = 0; d < st.nsum; ++d) {
    char ch = sum[d];
    st.sdim[d] = p.dims[(int)ch];
    st.as_s[d] = stride_of(p, A.idx, ch);
    st.bs_s[d] = B ? stride_of(p, B->idx, ch) : 0;
    st.sum_size *= st.sdim[d];
  }
  return st;
}

// order letters of `set` : first those of `pref` in pref order, then the rest in `base` order
std::string order_letters(const std::string& set, const std::string& pref, const std::string& base) {
  std::string r;
  for (char c : pref)
    if (set.find(c) != std::string::npos && r.find(c) == std::string::npos) r.push_back(c);
  for (char c : base)
    if (set.find(c) != std::string::npos && r.find(c) == std::string::npos) r.push_back(c);
  for (char c : set)
    if (r.find(c) == std::string::npos) r.push_back(c);
  return r;
}

// Greedy pairwise contraction of `ins` into `out_idx`.  If `target` is given the result is
// written there; otherwise a pure alias of a single matching input is allowed.
EinProgram compile_einsum(const Plan& p, std::vector<Operand> ins, const std::string& out_idx, Bump& bump,
                          const BufRef* target) {
  EinProgram prog;
  prog.result_idx = out_idx;
  std::string base = p.model;
  while (ins.size() > 1) {
    int bi = -1, bj = -1;
    double best = 1e300, best_macs = 1e300;
    std::string best_keep;
    for (size_t i = 0; i < ins.size(); ++i)
      for (size_t j = i + 1; j < ins.size(); ++j) {
        std::string needed = out_idx;
        for (size_t k = 0; k < ins.size(); ++k)
          if (k != i && k != j) needed += ins[k].idx;
        std::string uni = ins[i].idx;
        for (char c : ins[j].idx)
          if (uni.find(c) == std::string::npos) uni.push_back(c);
        std::string keep;
        for (char c : uni)
          if (needed.find(c) != std::string::npos) keep.push_back(c);
        double sz = (double)prod_idx(p, keep);
        double macs = (double)prod_idx(p, uni);
        if (sz < best || (sz == best && macs < best_macs)) {
          best = sz;
          best_macs = macs;
          bi = (int)i;
          bj = (int)j;
          best_keep = keep;
        }
      }
    std::string cidx = order_letters(best_keep, out_idx, base);
    BufRef c;
    c.kind = BUF_WS;
    c.elems = prod_idx(p, cidx);
    c.id = bump.take(c.elems * 4);
    EinStep st = make_step(p, ins[bi], &ins[bj], cidx, c);
    prog.macs += (double)st.out_size * (double)st.sum_size;
    prog.steps.push_back(st);
    Operand r{c, cidx};
    ins.erase(ins.begin() + bj);
    ins.erase(ins.begin() + bi);
    ins.push_back(r);
  }
  Operand& last = ins[0];
  if (last.idx == out_idx) {
    if (!target) {
      prog.result = last.buf;
      return prog;
    }
    if (!prog.steps.empty() && prog.steps.back().c.id == last.buf.id && last.buf.kind == BUF_WS) {
      prog.steps.back().c = *target;   // write the final pairwise step straight into the target
      prog.result = *target;
      return prog;
    }
  }
  BufRef c;
  if (target) {
    c = *target;
  } else {
    c.kind = BUF_WS;
    c.elems = prod_idx(p, out_idx);
    c.id = bump.take(c.elems * 4);
  }
  EinStep st = make_step(p, last, nullptr, out_idx, c);
  prog.macs += (double)st.out_size * (double)st.sum_size;
  prog.steps.push_back(st);
  prog.result = c;
  return prog;
}

BufRef factor_buf(const Plan& p, int l) {
  BufRef b;
  b.kind = BUF_FACTOR;
  b.id = l;
  b.elems = prod_idx(p, p.ops[l]);
  return b;
}

// Try one lowering candidate; returns false if invalid.
bool lower_candidate(const Plan& p, int ell, unsigned rowmask, unsigned pure_assign, Lowering& L, std::string& why) {
  const int M = (int)p.out.size();
  const int Lf = (int)p.ops.size();
  L = Lowering();
  L.ell = ell;
  std::vector<int> side(Lf, -1);   // 0 row, 1 col
  int pure_k = 0;
  for (int f = 0; f < Lf; ++f) {
    bool any_row = false, any_col = false;
    for (char c : p.ops[f]) {
      size_t m = p.out.find(c);
      if (m == std::string::npos) continue;
      if (rowmask >> m & 1u) any_row = true; else any_col = true;
    }
    if (any_row && any_col) { why = "straddle"; return false; }
    if (any_row) side[f] = 0;
    else if (any_col) side[f] = 1;
    else side[f] = (pure_assign >> pure_k++) & 1u;
  }
  if (side[ell] != 0) { why = "ell not on row side"; return false; }
  for (int m = 0; m < M; ++m) {
    if (rowmask >> m & 1u) { L.row_modes.push_back(m); L.row_idx.push_back(p.out[m]); }
    else { L.col_modes.push_back(m); L.col_idx.push_back(p.out[m]); }
  }
  for (int f = 0; f < Lf; ++f) (side[f] == 0 ? L.row_factors : L.col_factors).push_back(f);
  // bond: contracted letters present on both sides, in first-appearance order
  std::string rowl, coll;
  for (int f : L.row_factors) rowl += p.ops[f];
  for (int f : L.col_factors) coll += p.ops[f];
  for (char c : p.model) {
    if (!is_letter(c) || p.out.find(c) != std::string::npos) continue;
    if (rowl.find(c) != std::string::npos && coll.find(c) != std::string::npos && L.bond.find(c) == std::string::npos)
      L.bond.push_back(c);
  }
  L.K = prod_idx(p, L.bond);
  L.n_rows = prod_idx(p, L.row_idx);
  L.n_cols = prod_idx(p, L.col_idx);
  // Y strides of every mode (local shape)
  std::vector<int64_t> ys(M, 1);
  for (int m = M - 2; m >= 0; --m) ys[m] = ys[m + 1] * p.shape[m + 1];
  for (size_t k = 0; k < L.row_modes.size(); ++k) {
    L.rdim[k] = p.shape[L.row_modes[k]];
    L.rystride[k] = ys[L.row_modes[k]];
  }
  for (size_t k = 0; k < L.col_modes.size(); ++k) {
    L.cdim[k] = p.shape[L.col_modes[k]];
    L.cystride[k] = ys[L.col_modes[k]];
  }
  L.row_fast = (rowmask >> (M - 1)) & 1u;
  return true;
}

void build_tables(const Plan& p, Lowering& L, Bump& bump, bool merge);
void direct_run(Lowering& L);
void tc_geometry(const Plan& p, Lowering& L);
void finish_workspace(const Plan& p, Lowering& L, Bump& bump, const std::string& uidx);

// Fill programs, tables and workspace of a chosen candidate.
void finish_lowering(const Plan& p, Lowering& L, Bump& bump) {
  // U[row, bond] from the row-side factors
  std::vector<Operand> rin;
  for (int f : L.row_factors) rin.push_back({factor_buf(p, f), p.ops[f]});
  std::string uidx = L.row_idx + L.bond;
  L.uprog = compile_einsum(p, rin, uidx, bump, nullptr);
  build_tables(p, L, bump, false);
  // tcgen05 geometry first (the direct-V analysis needs the column blocks)
  tc_geometry(p, L);
  if (L.tc_ok) {
    direct_run(L);
    // no direct-V run with the component tables: merge every column factor into ONE table
    // over all column modes (consecutive rows for every tile) when that table is small
    // (L2-resident; its generation is a few microseconds)
    if (L.vd_tab < 0 && L.tabs.size() >= 1 && L.n_cols * L.K <= ((int64_t)8 << 20)) {
      build_tables(p, L, bump, true);
      direct_run(L);
    }
  }
  if (L.vd_tab >= 0) {
    L.vd_Kp = (L.K + 3) / 4 * 4;
    if (L.vd_Kp != L.K) L.ws_vpad = bump.take(L.vd_rows * L.vd_Kp * 4 + 256);
  }
  finish_workspace(p, L, bump, uidx);
}

// Column tables: connected components of the column factors via non-bond contracted letters,
// or (merge) one table over all column factors.
void build_tables(const Plan& p, Lowering& L, Bump& bump, bool merge) {
  L.tabs.clear();
  L.tabs_merged = merge;
  std::vector<int> comp(L.col_factors.size(), -1);
  int ncomp = 0;
  if (merge) {
    for (auto& c : comp) c = 0;
    ncomp = L.col_factors.empty() ? 0 : 1;
  }
  for (size_t i = 0; i < L.col_factors.size(); ++i) {
    if (comp[i] >= 0) continue;
    comp[i] = ncomp;
    bool grew = true;
    while (grew) {
      grew = false;
      for (size_t a = 0; a < L.col_factors.size(); ++a) {
        if (comp[a] != ncomp) continue;
        for (size_t b = 0; b < L.col_factors.size(); ++b) {
          if (comp[b] >= 0) continue;
          for (char c : p.ops[L.col_factors[a]]) {
            if (p.out.find(c) != std::string::npos || L.bond.find(c) != std::string::npos) continue;
            if (p.ops[L.col_factors[b]].find(c) != std::string::npos) { comp[b] = ncomp; grew = true; break; }
          }
        }
      }
    }
    ++ncomp;
  }
  // the kernels take at most kMaxTabs column tables: merge the two smallest components (their
  // outer product becomes one table) until the count fits
  while (ncomp > kMaxTabs) {
    std::vector<double> sz(ncomp, 1.0);
    for (int cidx = 0; cidx < ncomp; ++cidx) {
      std::string letters;
      for (size_t i = 0; i < L.col_factors.size(); ++i)
        if (comp[i] == cidx) letters += p.ops[L.col_factors[i]];
      std::string seen;
      for (char c : letters) {
        if (seen.find(c) != std::string::npos) continue;
        seen.push_back(c);
        if (L.col_idx.find(c) != std::string::npos || L.bond.find(c) != std::string::npos) sz[cidx] *= (double)p.dims[(int)c];
      }
    }
    int s0 = 0, s1 = 1;
    if (sz[s1] < sz[s0]) std::swap(s0, s1);
    for (int cidx = 2; cidx < ncomp; ++cidx) {
      if (sz[cidx] < sz[s0]) { s1 = s0; s0 = cidx; }
      else if (sz[cidx] < sz[s1]) s1 = cidx;
    }
    const int keep = std::min(s0, s1), gone = std::max(s0, s1);
    for (auto& c : comp) {
      if (c == gone) c = keep;
      else if (c > gone) --c;
    }
    --ncomp;
  }
  for (int cidx = 0; cidx < ncomp; ++cidx) {
    std::vector<Operand> cin;
    std::string letters;
    for (size_t i = 0; i < L.col_factors.size(); ++i)
      if (comp[i] == cidx) {
        cin.push_back({factor_buf(p, L.col_factors[i]), p.ops[L.col_factors[i]]});
        letters += p.ops[L.col_factors[i]];
      }
    std::string tidx;
    for (char c : L.col_idx)
      if (letters.find(c) != std::string::npos) tidx.push_back(c);
    for (char c : L.bond)
      if (letters.find(c) != std::string::npos) tidx.push_back(c);
    ColTable T;
    T.idx = tidx;
    T.prog = compile_einsum(p, cin, tidx, bump, nullptr);
    for (size_t k = 0; k < L.col_modes.size(); ++k) T.cstride[k] = stride_of(p, tidx, p.out[L.col_modes[k]]);
    T.boff.assign((size_t)L.K, 0);
    for (int64_t b = 0; b < L.K; ++b) {
      int64_t rem = b, off = 0;
      for (int d = (int)L.bond.size() - 1; d >= 0; --d) {
        int64_t n = p.dims[(int)L.bond[d]];
        off += (rem % n) * stride_of(p, tidx, L.bond[d]);
        rem /= n;
      }
      T.boff[(size_t)b] = (int32_t)off;
    }
    L.tabs.push_back(T);
  }
}

// Direct-V analysis (see Lowering::vd_tab): the longest trailing run of column modes that one
// table stores as consecutive rows of pitch K while the other tables are constant over it.
void direct_run(Lowering& L) {
  L.vd_tab = -1;
  L.vd_E = 0;
  const int nc = (int)L.col_modes.size();
  if (nc == 0 || L.tabs.empty()) return;
  const int64_t blk = L.tc_layout == 0 ? L.n_cols : L.tc_CI;
  for (size_t q = 0; q < L.tabs.size(); ++q) {
    const ColTable& T = L.tabs[q];
    bool unit = true;
    for (int64_t b = 0; b < L.K; ++b) unit &= T.boff[(size_t)b] == b;
    if (!unit) continue;
    int64_t want = L.K, E = 1;
    int m = nc;
    for (int d = nc - 1; d >= 0; --d) {
      bool ok = T.cstride[d] == want;
      for (size_t q2 = 0; q2 < L.tabs.size() && ok; ++q2)
        if (q2 != q) ok = L.tabs[q2].cstride[d] == 0;
      if (!ok) break;
      want *= L.cdim[d];
      E *= L.cdim[d];
      m = d;
    }
    if (m == nc) continue;
    // no 64-column tile may straddle two runs: tiles are 64-aligned inside each column block
    // (layout 0 / 1: one block of n_cols / CI columns; layout 2: CO blocks of CI columns)
    bool fits;
    if (L.tc_layout == 2) fits = (E % 64 == 0 && L.tc_CI % 64 == 0) || E % L.tc_CI == 0;
    else fits = E % 64 == 0 || E == blk;
    if (!fits) continue;
    L.vd_tab = (int)q;
    L.vd_E = E;
    L.vd_rows = T.prog.result.elems / L.K;
    return;
  }
}

// tcgen05 / TMA geometry: the row modes must be one adjacent block of Y modes; the column
// modes then split into an outer block (before) and an inner block (after).
void tc_geometry(const Plan& p, Lowering& L) {
  L.tc_ok = false;
  bool adjacent = !L.row_modes.empty();
  for (size_t k = 1; k < L.row_modes.size(); ++k) adjacent &= L.row_modes[k] == L.row_modes[k - 1] + 1;
  // bonds below one MMA K step (8) would be mostly zero padding on the tensor core and carry the
  // least averaging of its TF32 rounding (R26): they stay on the fp32 FFMA path
  if (adjacent && L.K >= 8 && L.K <= 64 && !L.col_modes.empty()) {
    const int M = (int)p.out.size();
    int r0 = L.row_modes.front(), r1 = L.row_modes.back();
    int64_t R = 1, CI = 1, CO = 1;
    for (int m = r0; m <= r1; ++m) R *= p.shape[m];
    for (int m = r1 + 1; m < M; ++m) CI *= p.shape[m];
    for (int m = 0; m < r0; ++m) CO *= p.shape[m];
    bool has_inner = r1 + 1 < M, has_outer = r0 > 0;
    L.tc_R = R;
    L.tc_CI = CI;
    L.tc_CO = CO;
    L.tc_rstride = CI;
    L.tc_costride = R * CI;
    L.tc_layout = !has_inner ? 0 : (has_outer ? 2 : 1);
    L.tc_KB = L.K <= 32 ? 32 : 64;
    // TMA: every non-innermost global stride must be a multiple of 16 bytes: 4 elements for
    // Y (fp32), 16 for the uint8 mask (a masked problem needs both)
    bool ok = true;
    auto strides_ok = [&](int64_t q) {
      if (L.tc_layout == 0) return R % q == 0;                      // stride of the column dim = R
      if (L.tc_layout == 1) return CI % q == 0;
      return CI % q == 0 && (R * CI) % q == 0;
    };
    ok = strides_ok(4);
    L.tc_mask_ok = strides_ok(16);
    // useful width: at least half of every 64-wide column box / 128-row box must be real data
    if (L.tc_layout == 0) ok = ok && R >= 64 && CO >= 32;
    else ok = ok && CI >= 32 && R >= 64;
    // TF32 operand rounding (R26): an entry of factor ell's numerator / denominator sums the Y
    // entries of its slab (Y with ell's observed indices fixed), whose RN errors (<= 2^-11
    // relative each) average as 1/sqrt(slab); small slabs stay on the fp32 FFMA path
    {
      int64_t slab = 1;
      for (size_t m = 0; m < p.out.size(); ++m)
        if (p.ops[L.ell].find(p.out[m]) == std::string::npos) slab *= p.shape[m];
      ok = ok && slab >= kTcMinSlab;
    }
    if (ok) {
      L.tc_ok = true;
      L.tc_row_blocks = (R + 127) / 128;
      L.tc_tiles = (L.tc_layout == 0) ? (CO + 63) / 64 : ((CI + 63) / 64) * (L.tc_layout == 2 ? CO : 1);
      // one CTA per SM (TMEM 512 columns, ~220 KB smem): never exceed one wave
      int64_t ch = std::max<int64_t>(1, p.num_sms / L.tc_row_blocks);
      ch = std::min(ch, L.tc_tiles);
      L.tc_chunks = ch;
      const int64_t tpc = (L.tc_tiles + ch - 1) / ch;
      L.tc_groups = std::max<int64_t>(1, (tpc + kDrainTiles - 1) / kDrainTiles);
    }
  }
}

// Workspace of the streaming pass and the epilogue program.
void finish_workspace(const Plan& p, Lowering& L, Bump& bump, const std::string& uidx) {
  // workspace for the streaming pass
  const int64_t BM = 64, BN = 64;
  int64_t row_blocks = (L.n_rows + BM - 1) / BM;
  int64_t col_tiles = (L.n_cols + BN - 1) / BN;
  int64_t target = (int64_t)p.num_sms * 4;
  int64_t chunks = std::max<int64_t>(1, (target + row_blocks - 1) / row_blocks);
  chunks = std::min(chunks, col_tiles);
  int64_t qelems = L.n_rows * L.K;
  while (chunks > 1 && chunks * qelems * 8 > (int64_t)512 << 20) chunks /= 2;
  L.n_chunks = chunks;
  L.ws_boff = bump.take((int64_t)L.tabs.size() * L.K * 4);
  L.ws_Qpart = bump.take(chunks * qelems * 2 * 4);
  L.ws_Q = bump.take(qelems * 2 * 4);
  int64_t felems = prod_idx(p, p.ops[L.ell]);
  L.ws_num = bump.take(2 * felems * 4);   // num | den adjacent (one all-reduce)
  L.ws_den = L.ws_num + felems * 4;
  L.ws_losspart = bump.take(row_blocks * chunks * 48);   // [3 roles] loss sums + counts (split fits)
  // epilogue: Num (ell's layout) = einsum(Q[row_idx + bond], row factors except ell)
  std::string qidx = uidx;
  if (L.row_factors.size() == 1 && p.ops[L.ell] == qidx) {
    L.epi_identity = true;
  } else {
    BufRef qa;
    qa.kind = BUF_WS;
    qa.id = L.ws_Q;
    qa.elems = qelems;
    std::vector<Operand> ein;
    ein.push_back({qa, qidx});
    for (int f : L.row_factors)
      if (f != L.ell) ein.push_back({factor_buf(p, f), p.ops[f]});
    BufRef tgt;
    tgt.kind = BUF_WS;
    tgt.id = L.ws_num;
    tgt.elems = felems;
    L.epi = compile_einsum(p, ein, p.ops[L.ell], bump, &tgt);
  }
  if (L.tc_ok) {
    L.ws_tc_Qpart = bump.take(L.tc_chunks * L.tc_groups * L.tc_row_blocks * 128 * L.K * 2 * 4);
    int64_t nparts = L.tc_row_blocks * L.tc_chunks;
    L.ws_tc_losspart = bump.take(nparts * 48);   // [3 roles] loss sums + counts (split fits)
  }
  L.ws_end = bump.off;
}

// Cost in MAC-equivalents: streamed MACs + column-operand generation + 8 x bytes moved
// through HBM by the side operands, split partials, reduction and tables.
double candidate_cost(const Plan& p, const Lowering& L) {
  double N = (double)p.n_local;
  double kp = (double)std::max<int64_t>(16, (L.K + 15) / 16 * 16);
  // the tcgen05 kernel streams at ~0.6 of HBM speed where the CUDA-core one does ~0.05-0.1
  // (profiles/): a lowering with a TMA geometry is preferred by that ratio
  double fused = N * 3.0 * kp * (L.tc_ok ? 0.125 : 1.0);
  double vgen = N / 64.0 * (double)L.K * (double)std::max<size_t>(1, L.tabs.size());
  double q = (double)L.n_rows * (double)L.K;
  double bytes = q * 4.0 * 2.0                              // U written + read
                 + (double)L.n_chunks * q * 8.0 * 2.0       // Q partials written + read
                 + q * 8.0 * 2.0;                           // Q written + read by the epilogue
  for (auto& t : L.tabs) bytes += 8.0 * (double)t.prog.result.elems;
  return fused + vgen + 8.0 * bytes;
}

}  // namespace

// Side-operand reuse inside one sweep (factor updates ell = 0, 1, ... in order): a program of
// update ell (its U or a column table) need not run when an earlier update e of the same sweep
// computed the same contraction (same steps over the same factors, same result layout), none
// of its input factors was updated in e .. ell - 1 (update m rewrites factor m only), and no
// workspace region of the updates e + 1 .. ell (other than the skipped program's own) overlaps
// the region holding e's result: update ell then reads that region.  c2: update 3's U (ijc) is
// update 2's table; c4: update 1's table (tdl) is update 0's, updates 3 and 4 use update 2's
// ijl.  The values are the floats the skipped launches would write (same kernels, same
// inputs), so results are bit-identical.
static bool prog_sem(const EinProgram& pr, std::string& sig, std::vector<int>& fac, std::vector<int64_t>& made) {
  std::ostringstream o;
  auto ref = [&](const BufRef& b) -> bool {
    if (b.kind == BUF_FACTOR) { fac.push_back((int)b.id); o << 'F' << b.id; return true; }
    if (b.kind == BUF_NONE) { o << '-'; return true; }
    const auto it = std::find(made.begin(), made.end(), b.id);
    if (it == made.end()) return false;   // reads a region it did not write: never reused
    o << '#' << (it - made.begin());
    return true;
  };
  for (const auto& st : pr.steps) {
    if (!ref(st.a) || !ref(st.b)) return false;
    o << ',' << st.a_idx << ',' << st.b_idx << ',' << st.c_idx << ';';
    made.push_back(st.c.id);
  }
  o << '>' << pr.result_idx << ':' << pr.result.elems;
  sig = o.str();
  return !pr.steps.empty() && pr.result.kind == BUF_WS && pr.steps.back().c.id == pr.result.id;
}
void sweep_reuse(Plan& p) {
  const int L = (int)p.low.size();
  struct Done { std::string sig; std::vector<int> fac; BufRef where; };
  std::vector<std::vector<Done>> done(L);   // per update: its programs and where their results are
  for (int ell = 0; ell < L; ++ell) {
    Lowering& cur = p.low[ell];
    cur.reuse_u = false;
    cur.reuse_tab.assign(cur.tabs.size(), 0);
    cur.alias_tab.assign(cur.tabs.size(), BufRef{});
    for (int q = -1; q < (int)cur.tabs.size(); ++q) {
      const EinProgram& pr = q < 0 ? cur.uprog : cur.tabs[q].prog;
      std::string sig;
      std::vector<int> fac;
      std::vector<int64_t> own;
      if (!prog_sem(pr, sig, fac, own)) continue;
      BufRef where = pr.result;
      bool reused = false;
      for (int e = ell - 1; e >= 0 && !reused; --e) {
        for (const Done& d : done[e]) {
          if (d.sig != sig) continue;
          bool ok = true;
          for (int f : fac) ok = ok && (f < e || f >= ell);
          const int64_t r0 = d.where.id, r1 = d.where.id + d.where.elems * 4;
          for (int m = e + 1; m <= ell && ok; ++m)
            for (const auto& a : p.low[m].ws_allocs) {
              if (m == ell && std::find(own.begin(), own.end(), a.first) != own.end()) continue;
              ok = ok && (a.second <= r0 || a.first >= r1);
            }
          if (ok) { where = d.where; reused = true; }
          break;   // the nearest update that computed it decides
        }
        if (!done[e].empty() && !reused) {
          bool found = false;
          for (const Done& d : done[e]) found = found || d.sig == sig;
          if (found) break;
        }
      }
      if (reused) {
        if (q < 0) { cur.reuse_u = true; cur.alias_u = where; }
        else { cur.reuse_tab[q] = 1; cur.alias_tab[q] = where; }
      }
      done[ell].push_back({sig, fac, where});
    }
  }
}

int lower_all(Plan& p, std::string& err) {
  const int M = (int)p.out.size();
  const int Lf = (int)p.ops.size();
  int npure = 0;
  for (auto& op : p.ops) {
    bool anyobs = false;
    for (char c : op) anyobs |= p.out.find(c) != std::string::npos;
    if (!anyobs) ++npure;
  }
  if (npure > 6) { err = "too many purely-contracted factors"; return NEF_E_UNSUPPORTED; }
  p.low.assign(Lf, Lowering());
  int64_t ws = 0;
  for (int ell = 0; ell < Lf; ++ell) {
    Lowering best;
    double best_cost = 1e300;
    bool found = false;
    unsigned best_rm = 0, best_pa = 0;
    for (unsigned rm = 1; rm < (1u << M); ++rm) {
      for (unsigned pa = 0; pa < (1u << npure); ++pa) {
        Lowering cand;
        std::string why;
        if (!lower_candidate(p, ell, rm, pa, cand, why)) continue;
        if (cand.K > 64) continue;                        // both streaming kernels take bonds <= 64
        Bump tmp;
        finish_lowering(p, cand, tmp);
        double c = candidate_cost(p, cand) + cand.uprog.macs + cand.epi.macs;
        for (auto& t : cand.tabs) c += t.prog.macs;
        if (cand.n_rows * cand.K > ((int64_t)1 << 28)) c += 1e18;  // U must stay small
        if (rm == (1u << M) - 1) c += 1e17;                        // no columns: last resort
        if (c < best_cost) { best_cost = c; best = cand; found = true; best_rm = rm; best_pa = pa; }
      }
    }
    if (!found) {
      err = "no (row, col, bond) lowering with bond <= 64 for factor " + std::to_string(ell) + " ('" + p.ops[ell] + "')";
      return NEF_E_UNSUPPORTED;
    }
    // rebuild with a fresh bump so offsets are final
    Bump bump;
    Lowering L;
    std::string why;
    lower_candidate(p, ell, best_rm, best_pa, L, why);
    finish_lowering(p, L, bump);
    L.cost = best_cost;
    L.ws_allocs = bump.log;
    ws = std::max<int64_t>(ws, L.ws_end);
    p.low[ell] = std::move(L);
  }
  sweep_reuse(p);
  p.ws_trace = (ws + 255) / 256 * 256;
  // sentinel pass sums (R25): [data-only loss sum][observed count], then its block partials
  p.ws_dterm = p.ws_trace + (int64_t)8 * 4096;
  p.ws_dpart = p.ws_dterm + 256;
  // nef_fit_split: a copy of the factors entering each sweep (a stopped fit returns that iterate)
  p.ws_fsave = (p.ws_dpart + (int64_t)16 * (kSentParts) + 255) / 256 * 256;
  int64_t fbytes = 0;
  for (auto& sh : p.fshape) {
    int64_t n = 1;
    for (auto d : sh) n *= d;
    fbytes += (n * 4 + 255) / 256 * 256;
  }
  // split partials of GEMM-shaped einsum steps (side operands, epilogues): the largest need
  int64_t escr = 0;
  for (const auto& L : p.low) {
    for (const auto& st : L.uprog.steps) escr = std::max<int64_t>(escr, einstep_scratch_floats(st));
    for (const auto& t : L.tabs)
      for (const auto& st : t.prog.steps) escr = std::max<int64_t>(escr, einstep_scratch_floats(st));
    for (const auto& st : L.epi.steps) escr = std::max<int64_t>(escr, einstep_scratch_floats(st));
  }
  p.ws_escr = (p.ws_fsave + fbytes + 255) / 256 * 256;
  // NaN-sentinel copy of the local Y (nef_fit with a mask, R5): 4 B per local entry
  p.ws_sent = (p.ws_escr + escr * 4 + 255) / 256 * 256;
  p.ws_bytes = (size_t)(p.ws_sent + p.n_local * 4 + 256);
  return NEF_OK;
}

int build_plan(const char* einsum, int n_modes, const int64_t* shape, int n_ranks, const int64_t* ranks, Plan& p,
               std::string& err) {
  int st = parse_model(einsum, p.ops, p.out, err);
  if (st) return st;
  if (n_modes != (int)p.out.size()) { err = "shape has " + std::to_string(n_modes) + " dims, output has " + std::to_string(p.out.size()); return NEF_E_SHAPE; }
  if (n_modes > 0 && !shape) { err = "null shape"; return NEF_E_ARG; }
  std::memset(p.dims, 0, sizeof(p.dims));
  int64_t total = 1;
  for (int m = 0; m < n_modes; ++m) {
    if (shape[m] <= 0) { err = "non-positive dimension"; return NEF_E_SHAPE; }
    p.dims[(int)p.out[m]] = shape[m];
    if (mul_overflow(total, shape[m], &total)) { err = "number of entries overflows int64"; return NEF_E_SHAPE; }
  }
  std::string contracted;
  for (auto& op : p.ops)
    for (char c : op)
      if (p.out.find(c) == std::string::npos && contracted.find(c) == std::string::npos) contracted.push_back(c);
  if (n_ranks != (int)contracted.size()) {
    err = "expected " + std::to_string(contracted.size()) + " contracted-index sizes, got " + std::to_string(n_ranks);
    return NEF_E_SHAPE;
  }
  if (n_ranks > 0 && !ranks) { err = "null ranks"; return NEF_E_ARG; }
  for (int k = 0; k < n_ranks; ++k) {
    if (ranks[k] <= 0) { err = "non-positive rank"; return NEF_E_SHAPE; }
    p.dims[(int)contracted[k]] = ranks[k];
  }
  p.model.clear();
  for (size_t l = 0; l < p.ops.size(); ++l) p.model += (l ? "," : "") + p.ops[l];
  p.model += "->" + p.out;
  // einstr_l = swap(model_str, l)
  p.einstr.clear();
  for (size_t l = 0; l < p.ops.size(); ++l) {
    std::string s;
    for (size_t k = 0; k < p.ops.size(); ++k) s += (k ? "," : "") + (k == l ? p.out : p.ops[k]);
    p.einstr.push_back(s + "->" + p.ops[l]);
  }
  p.gshape.assign(shape, shape + n_modes);
  p.shape = p.gshape;
  p.n_local = total;
  p.local_begin = 0;
  p.local_len = n_modes ? p.shape[0] : 1;
  p.shard_mode = -1;
  p.factor_has_shard.assign(p.ops.size(), false);
  return relower(p, err);
}

int relower(Plan& p, std::string& err) {
  int64_t total = 1;
  for (auto d : p.shape) total *= d;
  p.n_local = total;
  // local factor shapes
  int64_t saved = 0;
  if (p.shard_mode >= 0) {
    saved = p.dims[(int)p.out[p.shard_mode]];
    p.dims[(int)p.out[p.shard_mode]] = p.shape[p.shard_mode];
  }
  p.fshape.clear();
  for (auto& op : p.ops) {
    std::vector<int64_t> s;
    for (char c : op) s.push_back(p.dims[(int)c]);
    p.fshape.push_back(s);
  }
  (void)saved;   // dims keep the LOCAL size of the shard mode: the plan describes this rank
  return lower_all(p, err);
}

static void json_prog(std::ostringstream& o, const EinProgram& pr) {
  o << "{\"steps\":[";
  for (size_t i = 0; i < pr.steps.size(); ++i) {
    const EinStep& s = pr.steps[i];
    auto br = [&](const BufRef& b) {
      std::ostringstream t;
      if (b.kind == BUF_FACTOR) t << "\"F" << b.id << "\"";
      else if (b.kind == BUF_WS) t << "\"W" << b.id << "\"";
      else t << "null";
      return t.str();
    };
    o << (i ? "," : "") << "{\"a\":" << br(s.a) << ",\"a_idx\":\"" << s.a_idx << "\",\"b\":" << br(s.b)
      << ",\"b_idx\":\"" << s.b_idx << "\",\"c\":" << br(s.c) << ",\"c_idx\":\"" << s.c_idx << "\"}";
  }
  auto br = [&](const BufRef& b) {
    std::ostringstream t;
    if (b.kind == BUF_FACTOR) t << "\"F" << b.id << "\"";
    else if (b.kind == BUF_WS) t << "\"W" << b.id << "\"";
    else t << "null";
    return t.str();
  };
  o << "],\"result\":" << br(pr.result) << ",\"result_idx\":\"" << pr.result_idx << "\",\"macs\":" << pr.macs << "}";
}

std::string describe_plan(const Plan& p) {
  std::ostringstream o;
  o << "{\"model\":\"" << p.model << "\",\"einstr\":[";
  for (size_t l = 0; l < p.einstr.size(); ++l) o << (l ? "," : "") << "\"" << p.einstr[l] << "\"";
  o << "],\"shape\":[";
  for (size_t m = 0; m < p.shape.size(); ++m) o << (m ? "," : "") << p.shape[m];
  o << "],\"shard_mode\":" << p.shard_mode << ",\"rank\":" << p.rank << ",\"world\":" << p.world
    << ",\"local_begin\":" << p.local_begin << ",\"local_len\":" << p.local_len << ",\"factor_has_shard\":[";
  for (size_t l = 0; l < p.factor_has_shard.size(); ++l) o << (l ? "," : "") << (p.factor_has_shard[l] ? "true" : "false");
  o << "],\"workspace_bytes\":" << p.ws_bytes << ",\"lowerings\":[";
  for (size_t l = 0; l < p.low.size(); ++l) {
    const Lowering& L = p.low[l];
    o << (l ? "," : "") << "{\"ell\":" << L.ell << ",\"row_idx\":\"" << L.row_idx << "\",\"col_idx\":\"" << L.col_idx
      << "\",\"bond\":\"" << L.bond << "\",\"K\":" << L.K << ",\"n_rows\":" << L.n_rows << ",\"n_cols\":" << L.n_cols
      << ",\"row_fast\":" << (L.row_fast ? "true" : "false") << ",\"n_chunks\":" << L.n_chunks
      << ",\"tc\":" << (L.tc_ok ? "true" : "false") << ",\"tc_mask_ok\":" << (L.tc_mask_ok ? "true" : "false") << ",\"tc_layout\":" << L.tc_layout << ",\"tc_R\":" << L.tc_R
      << ",\"tc_CI\":" << L.tc_CI << ",\"tc_CO\":" << L.tc_CO << ",\"tc_KB\":" << L.tc_KB
      << ",\"tc_tiles\":" << L.tc_tiles << ",\"tc_chunks\":" << L.tc_chunks << ",\"tc_groups\":" << L.tc_groups << ",\"vd_tab\":" << L.vd_tab << ",\"vd_E\":" << L.vd_E << ",\"tabs_merged\":" << (L.tabs_merged ? "true" : "false") << ",\"row_factors\":[";
    for (size_t k = 0; k < L.row_factors.size(); ++k) o << (k ? "," : "") << L.row_factors[k];
    o << "],\"col_factors\":[";
    for (size_t k = 0; k < L.col_factors.size(); ++k) o << (k ? "," : "") << L.col_factors[k];
    o << "],\"U\":";
    json_prog(o, L.uprog);
    o << ",\"tables\":[";
    for (size_t t = 0; t < L.tabs.size(); ++t) {
      o << (t ? "," : "") << "{\"idx\":\"" << L.tabs[t].idx << "\",\"prog\":";
      json_prog(o, L.tabs[t].prog);
      o << "}";
    }
    o << "],\"Q\":\"W" << L.ws_Q << "\",\"epi_identity\":" << (L.epi_identity ? "true" : "false") << ",\"epi\":";
    json_prog(o, L.epi);
    o << ",\"reuse_u\":" << (L.reuse_u ? "true" : "false") << ",\"reuse_tab\":[";
    for (size_t q = 0; q < L.reuse_tab.size(); ++q) o << (q ? "," : "") << (L.reuse_tab[q] ? "true" : "false");
    o << "],\"cost\":" << L.cost << "}";
  }
  o << "]}";
  return o.str();
}

}  // namespace nef
