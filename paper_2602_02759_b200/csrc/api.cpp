// C ABI of libnef (include/nef.h): orchestration of Algorithm 1 on the device.
//
// Per factor update ell (Alg. 1 lines 6-9):
//   1. side operands  U = einsum(row factors -> rows,bond), column tables     (small-einsum engine)
//   2. fused pass     Q_a = a(Y, U V^T) V, Q_b = b(Y, U V^T) V, one read of Y / mask
//   3. reduce         fixed-order sum of split-column partials
//   4. epilogue       A = einsum(swap(rowmodel, ell)) with Q_a (B likewise)   (= einstr_ell)
//   5. [sharded]      ncclAllReduce(A|B) for factors without the shard mode
//   6. update         Theta <- max(eps, Theta * g^{-1}(A/B))
// The loss of the iterate entering a sweep is accumulated inside the first factor's fused
// pass; one extra loss-only pass gives the final trace entry.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.h"
#include "kernels_tc.h"
#include "nef_internal.h"
#include "../../include/nef.h"

// A captured sweep of nef_fit (CUDA graph, replayed once per sweep; see sweep_graph below)
struct SweepGraph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::string key;                         // the inputs it was captured for (pointers, loss, flags)
  std::vector<cudaGraphNode_t> ev_nodes;   // event-record nodes of the streaming launches, in order
  std::vector<cudaEvent_t> own;            // the events they record when profiling is off
  std::vector<double> bytes;               // algorithmic bytes of each streaming launch
  bool on_prof = false;                    // nodes currently point at profiling events
  ~SweepGraph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    for (auto e : own) cudaEventDestroy(e);
  }
};

struct nef_plan_s {
  nef::Plan p;
  SweepGraph* g = nullptr;            // cached sweep graph (one entry: the last input set)
  cudaStream_t cap_stream = nullptr;  // private stream the sweep is captured on (the caller's may be
                                      // the legacy default stream, which cannot be captured)
  bool graph_failed = false;          // a capture failed: this plan launches kernel by kernel
  ~nef_plan_s() {
    delete g;
    if (cap_stream) cudaStreamDestroy(cap_stream);
  }
};

namespace {

thread_local std::string g_err;
thread_local int64_t g_launches = 0;
int g_policy = 0;
float* g_debug = nullptr;   // optional device dump of the tcgen05 kernel's first tile (tests)
long long* g_trace = nullptr;   // optional pipeline timeline of the tcgen05 kernel (diagnostics)
bool g_no_memo = std::getenv("NEF_NO_REUSE") != nullptr;        // diagnostics: recompute every side operand
bool g_no_sentinel = std::getenv("NEF_NO_SENTINEL") != nullptr;   // diagnostics: stream the uint8 mask
bool g_no_lconst = std::getenv("NEF_NO_LCONST") != nullptr;     // diagnostics: loss passes compute the whole divergence (R25 off)
bool g_no_sqy = std::getenv("NEF_NO_SQY") != nullptr;           // diagnostics: (0.5, 0) streams y, not sqrt(y)
// diagnostics: NEF_TC_VDIRECT=0 generates V per tile instead of TMA-loading direct-V table rows
bool g_vdirect = [] { const char* e = std::getenv("NEF_TC_VDIRECT"); return !e || std::atoi(e) != 0; }();

bool g_graphs = [] { const char* e = std::getenv("NEF_NO_GRAPH"); return !e || e[0] != '1'; }();   // diagnostics

// live CUDA-event timing of the streaming kernel (nef_profile_*)
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> ev;   // pairs (start, end)
  size_t used = 0;               // number of pairs recorded since enable
  double bytes = 0;
  SweepGraph* cap = nullptr;     // a sweep graph being captured: its own events, as graph nodes
};
Prof g_prof;

bool prof_reserve() {
  if (2 * g_prof.used + 2 > g_prof.ev.size()) {
    for (int k = 0; k < 64; ++k) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) { g_prof.on = false; return false; }
      g_prof.ev.push_back(e);
    }
  }
  return true;
}

void prof_begin(cudaStream_t s) {
  if (g_prof.cap) {   // capture: an external event-record node (re-pointed at every replay)
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_prof.cap->own.push_back(e);
    cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    return;
  }
  if (!g_prof.on || !prof_reserve()) return;
  cudaEventRecord(g_prof.ev[2 * g_prof.used], s);
}

void prof_end(cudaStream_t s, double bytes) {
  if (g_prof.cap) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    g_prof.cap->own.push_back(e);
    g_prof.cap->bytes.push_back(bytes);
    cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
    return;
  }
  if (!g_prof.on) return;
  cudaEventRecord(g_prof.ev[2 * g_prof.used + 1], s);
  g_prof.used++;
  g_prof.bytes += bytes;
}

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) return fail(NEF_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ------------------------------------------------------------------ NCCL (dlopen)
struct Uid {
  char internal[128];
};
struct Nccl {
  bool loaded = false;
  void* h = nullptr;
  int (*GetUniqueId)(void*) = nullptr;
  int (*CommInitRank)(void**, int, Uid, int) = nullptr;  // ncclUniqueId by value
  int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*CommDestroy)(void*) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};
Nccl g_nccl;

bool load_nccl(std::string& err) {
  if (g_nccl.loaded) return true;
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* n : names) {
    g_nccl.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    if (g_nccl.h) break;
  }
  if (!g_nccl.h) { err = std::string("cannot dlopen libnccl.so.2: ") + dlerror(); return false; }
  g_nccl.GetUniqueId = (int (*)(void*))dlsym(g_nccl.h, "ncclGetUniqueId");
  g_nccl.CommInitRank = (int (*)(void**, int, Uid, int))dlsym(g_nccl.h, "ncclCommInitRank");
  g_nccl.AllReduce = (int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t))dlsym(g_nccl.h, "ncclAllReduce");
  g_nccl.CommDestroy = (int (*)(void*))dlsym(g_nccl.h, "ncclCommDestroy");
  g_nccl.GetErrorString = (const char* (*)(int))dlsym(g_nccl.h, "ncclGetErrorString");
  if (!g_nccl.GetUniqueId || !g_nccl.CommInitRank || !g_nccl.AllReduce || !g_nccl.CommDestroy) {
    err = "libnccl is missing symbols";
    return false;
  }
  g_nccl.loaded = true;
  return true;
}
constexpr int kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclInt64 = 4, kNcclSum = 0;

// ------------------------------------------------------------------ run context
struct Ctx {
  const nef::Plan* p;
  float* const* F;
  char* ws;
  size_t ws_bytes;
  cudaStream_t s;
  const float* ysent = nullptr;   // NaN-sentinel copy of Y (mask folded in), when prepared
  const double* loff = nullptr;   // R25: [data-only loss sum][observed count] of the sentinel pass
  double lscale = 1.0;            //      loss = lscale * (streamed part) + loff[0]
  const float* aux = nullptr;     // per-entry phi / n (App. B losses), Y's layout; CUDA-core kernel only
  bool sqy = false;               // ysent holds sqrt(y) for the (0.5, 0) pair (R35), masked or not
  int split = 0;                  // the mask holds labels 0..3 (R29); loss slots are [3] per pass
  bool memo = false;              // inside a sweep run in update order: skip the side-operand
                                  // programs the planner marked as reusable (sweep_reuse)
  // split fits: after the loss-carrying pass, copy the loss slots to pinned host memory and
  // record an event, so the host can take the stopping decision while the sweep continues
  void* pin = nullptr;
  cudaEvent_t pin_ev = nullptr;
  bool pin_counts = false;
};

float* resolve(const Ctx& c, const nef::BufRef& b) {
  if (b.kind == nef::BUF_FACTOR) return c.F[b.id];
  if (b.kind == nef::BUF_WS) return reinterpret_cast<float*>(c.ws + b.id);
  return nullptr;
}

// run a program; `from`/`to` remap one workspace offset (used to run the epilogue on Q_b)
int run_prog(const Ctx& c, const nef::EinProgram& pr, int64_t from1 = -1, int64_t to1 = -1, int64_t from2 = -1,
             int64_t to2 = -1) {
  auto res = [&](nef::BufRef b) {
    if (b.kind == nef::BUF_WS) {
      if (b.id == from1) b.id = to1;
      else if (b.id == from2) b.id = to2;
    }
    return resolve(c, b);
  };
  for (const auto& st : pr.steps) {
    cudaError_t e = nef::launch_einstep(st, res(st.a), st.b.kind == nef::BUF_NONE ? nullptr : res(st.b), res(st.c), c.s,
                                        reinterpret_cast<float*>(c.ws + c.p->ws_escr));
    ++g_launches;
    if (e != cudaSuccess) return fail(NEF_E_CUDA, std::string("einstep: ") + cudaGetErrorString(e));
  }
  return NEF_OK;
}

const float* prog_result(const Ctx& c, const nef::EinProgram& pr) { return resolve(c, pr.result); }

// Fill FusedArgs for lowering L; U and tables must already be computed.
nef::FusedArgs fused_args(const Ctx& c, const nef::Lowering& L, const float* Y, const uint8_t* M, int mode,
                          const nef::DivParams& dv, std::vector<int32_t>& boff_host) {
  nef::FusedArgs a{};
  a.Y = Y;
  a.M = M;
  a.n_rows = L.n_rows;
  a.n_cols = L.n_cols;
  a.K = (int)L.K;
  a.nr = (int)L.row_modes.size();
  a.nc = (int)L.col_modes.size();
  for (int k = 0; k < a.nr; ++k) { a.rdim[k] = L.rdim[k]; a.rys[k] = L.rystride[k]; }
  for (int k = 0; k < a.nc; ++k) { a.cdim[k] = L.cdim[k]; a.cys[k] = L.cystride[k]; }
  a.U = (c.memo && L.reuse_u) ? resolve(c, L.alias_u) : prog_result(c, L.uprog);
  a.ntab = (int)L.tabs.size();
  boff_host.clear();
  for (int q = 0; q < a.ntab; ++q) {
    a.tab[q] = (c.memo && q < (int)L.reuse_tab.size() && L.reuse_tab[q]) ? resolve(c, L.alias_tab[q])
                                                                          : prog_result(c, L.tabs[q].prog);
    for (int k = 0; k < a.nc; ++k) a.tcs[q][k] = L.tabs[q].cstride[k];
    boff_host.insert(boff_host.end(), L.tabs[q].boff.begin(), L.tabs[q].boff.end());
  }
  a.boff = boff_host.data();   // host pointer: copied into kernel parameters at launch
  a.row_fast = L.row_fast ? 1 : 0;
  a.n_chunks = L.n_chunks;
  int64_t tiles = (L.n_cols + 63) / 64;
  a.tiles_per_chunk = (tiles + L.n_chunks - 1) / L.n_chunks;
  a.Qpart = reinterpret_cast<float*>(c.ws + L.ws_Qpart);
  a.losspart = reinterpret_cast<double*>(c.ws + L.ws_losspart);
  int64_t nparts = ((L.n_rows + 63) / 64) * L.n_chunks;
  a.countpart = reinterpret_cast<long long*>(c.ws + L.ws_losspart + 3 * nparts * 8);
  a.dv = dv;
  a.mode = mode;
  a.aux = c.aux;
  a.split = (c.split && M) ? 1 : 0;
  return a;
}

int side_operands(const Ctx& c, const nef::Lowering& L) {
  int st = (c.memo && L.reuse_u) ? NEF_OK : run_prog(c, L.uprog);
  if (st) return st;
  for (size_t q = 0; q < L.tabs.size(); ++q) {
    if (c.memo && q < L.reuse_tab.size() && L.reuse_tab[q]) continue;
    st = run_prog(c, L.tabs[q].prog);
    if (st) return st;
  }
  return NEF_OK;
}

// Where one streaming launch left its partials.
struct StreamOut {
  float* Qpart = nullptr;
  int64_t n_chunks = 1;
  double* losspart = nullptr;
  long long* countpart = nullptr;
  int64_t nparts = 0;
  bool lconst = false;            // loss partials hold only the factor-dependent part (R25)
};

// the tcgen05 kernel takes a per-entry parameter stream (NB phi_i / binomial n_i) as a second TMA
// ring next to the sentinel copy or unmasked Y (not next to a streamed uint8 mask)
bool use_tc(const nef::Lowering& L, const uint8_t* M, bool sentinel = false, const float* aux = nullptr,
            int kind = 0) {
  if (aux && (!(kind == nef::EW_NB || kind == nef::EW_BINOM) || (M && !sentinel) ||
              (reinterpret_cast<uintptr_t>(aux) & 15)))
    return false;
  return g_policy == 0 && L.tc_ok && (!M || sentinel || (L.tc_mask_ok && (reinterpret_cast<uintptr_t>(M) & 15) == 0));
}

// One streaming pass over Y (+mask) for lowering L: the tcgen05 kernel where the planner
// found a TMA geometry, else the CUDA-core kernel.  U and the column tables must be ready.
// TcArgs of one restart's pass; chunks_b > 0 forces the chunk count (batched restarts)
int fill_tc(const Ctx& c, const nef::Lowering& L, const nef::FusedArgs& a, const std::vector<int32_t>& boff, int mode,
            const nef::DivParams& dvk, bool sent, const uint8_t* M, int64_t chunks_b, nef::tc::TcArgs& t,
            int64_t& chunks, StreamOut& o) {
  t = nef::tc::TcArgs{};
  t.layout = L.tc_layout;
  t.R = L.tc_R;
  t.CI = L.tc_CI;
  t.CO = L.tc_CO;
  t.tiles_inner = (L.tc_CI + 63) / 64;
  t.tiles = L.tc_tiles;
  const int64_t want = chunks_b > 0 ? chunks_b : L.tc_chunks;
  int64_t tpc = (L.tc_tiles + want - 1) / want;
  chunks = (L.tc_tiles + tpc - 1) / tpc;   // no empty chunk
  t.tiles_per_chunk = tpc;
  t.K = (int)L.K;
  t.KB = L.tc_KB;
  t.n_rows = L.n_rows;
  t.U = a.U;
  t.nc = a.nc;
  for (int k = 0; k < a.nc; ++k) t.cdim[k] = a.cdim[k];
  t.ntab = a.ntab;
  for (int q = 0; q < a.ntab; ++q) {
    t.tab[q] = a.tab[q];
    for (int k = 0; k < a.nc; ++k) t.tcs[q][k] = a.tcs[q][k];
    for (int k = 0; k < L.K; ++k) t.boff[q][k] = boff[(size_t)q * L.K + k];
  }
  bool v4 = (L.K % 4 == 0);
  for (int q = 0; q < a.ntab && v4; ++q) {
    v4 = (reinterpret_cast<uintptr_t>(a.tab[q]) & 15) == 0;
    for (int k = 0; k < a.nc; ++k) v4 = v4 && (a.tcs[q][k] % 4 == 0);
    for (int k = 0; k < L.K; ++k) v4 = v4 && (boff[(size_t)q * L.K + k] == k);
  }
  t.vec4 = v4 && a.ntab > 0 ? 1 : 0;
  // direct V (planner: Lowering::vd_tab): the tile's V rows are consecutive rows of one
  // table, TMA-loaded; a K % 4 != 0 table is first copied to a 16-byte row pitch
  t.vdirect = 0;
  if (g_vdirect && L.vd_tab >= 0) {
    t.vdirect = 1;
    t.var_tab = L.vd_tab;
    t.var_rows = L.vd_rows;
    t.vd_E = L.vd_E;
    // tiles per run: runs are whole column blocks (E a multiple of the block extent, or
    // E == block) or E / 64 aligned tiles
    const int64_t blk = L.tc_layout == 0 ? L.tc_CO : L.tc_CI;
    const int64_t tiles_blk = (blk + 63) / 64;
    if (L.vd_E % blk == 0) t.vd_tpr = (L.vd_E / blk) * tiles_blk;
    else t.vd_tpr = L.vd_E / 64;
    t.vd_pitch = L.vd_Kp;
    t.vd_rows_ptr = a.tab[L.vd_tab];
    if (L.ws_vpad >= 0) {
      float* pad = reinterpret_cast<float*>(c.ws + L.ws_vpad);
      CK(nef::launch_pad_rows(a.tab[L.vd_tab], pad, L.vd_rows, L.K, L.vd_Kp, c.s));
      ++g_launches;
      t.vd_rows_ptr = pad;
    }
  }
  t.Qpart = reinterpret_cast<float*>(c.ws + L.ws_tc_Qpart);
  t.losspart = reinterpret_cast<double*>(c.ws + L.ws_tc_losspart);
  o.nparts = L.tc_row_blocks * chunks;
  t.countpart = reinterpret_cast<long long*>(c.ws + L.ws_tc_losspart + 3 * o.nparts * 8);
  t.dv = dvk;
  t.mode = mode;
  t.split = (c.split && M && !sent) ? 1 : 0;
  t.lconst = ((sent || !M) && c.loff && mode != 0) ? 1 : 0;
  // unmasked Y streamed as is: every entry is observed, so the kernel must not read "missing"
  // from a sign bit (an observed -0.0 is a zero); the sentinel copy canonicalises -0 itself
  t.absy = (!M && !sent) ? 1 : 0;
  t.debug = g_debug;
  t.trace = g_trace;
  t.n_groups = (tpc + nef::kDrainTiles - 1) / nef::kDrainTiles;
  o.Qpart = t.Qpart;
  o.n_chunks = chunks * t.n_groups;
  o.losspart = t.losspart;
  o.countpart = t.countpart;
  o.lconst = t.lconst != 0;
  return NEF_OK;
}

// One streaming pass over Y (+mask) for lowering L, for S restarts (contexts cs[0..S-1], N4): the
// tcgen05 kernel where the planner found a TMA geometry - ONE launch whose z index is the
// restart, so every restart's CTAs stream the same Y tiles (the other restarts' reads hit L2) -
// else the CUDA-core kernel per restart.  U and the column tables must be ready.
int stream_pass_multi(const Ctx* cs, int S, const nef::Lowering& L, const float* Y, const uint8_t* M, int mode,
                      const nef::DivParams& dv, StreamOut* os) {
  const Ctx& c = cs[0];
  // kernel limits (the planner keeps every lowering inside them; checked again before any launch)
  if (L.tabs.size() > (size_t)nef::kMaxTabs || L.K > 64)
    return fail(NEF_E_UNSUPPORTED, "lowering exceeds the kernels' limits (<= 4 column tables, bond <= 64)");
  std::vector<int32_t> boff;
  const double bytes = (double)c.p->n_local * ((M ? 5.0 : 4.0) + (c.aux ? 4.0 : 0.0));
  // split fits: the loss-carrying passes stream Y with the labels (train / validation / heldout
  // losses of one pass); update-only passes stream the train-folded sentinel copy
  const bool sent = c.ysent && (M || c.sqy) && !(c.split && mode != 0);
  nef::DivParams dvk = dv;
  if (use_tc(L, M, sent, c.aux, dv.kind) && (S == 1 || (g_vdirect && L.vd_tab >= 0))) {
    const float* Yk = Y;
    const uint8_t* Mk = M;
    if (sent) {   // stream the NaN-sentinel copy: no mask stream (4 B / entry)
      Yk = c.ysent;
      Mk = nullptr;
      if (c.sqy) dvk.kind = nef::EW_A05_B0_SQ;   // the copy holds sqrt(y) (R35)
    }
    // batched restarts: one wave of row blocks x chunks x restarts; the restarts' partials must
    // fit the single-restart workspace layout (else one launch per restart)
    int64_t chunks_b = 0;
    if (S > 1) {
      chunks_b = std::max<int64_t>(1, c.p->num_sms / (L.tc_row_blocks * S));
      const int64_t tpc = (L.tc_tiles + chunks_b - 1) / chunks_b;
      const int64_t groups = (tpc + nef::kDrainTiles - 1) / nef::kDrainTiles;
      if (chunks_b * groups > L.tc_chunks * L.tc_groups) {
        for (int r = 0; r < S; ++r)
          if (int st = stream_pass_multi(cs + r, 1, L, Y, M, mode, dv, os + r)) return st;
        return NEF_OK;
      }
    }
    nef::tc::TcArgs t0{};
    int64_t chunks = 0;
    for (int r = 0; r < S; ++r) {
      nef::FusedArgs a = fused_args(cs[r], L, Yk, Mk, mode, dv, boff);
      nef::tc::TcArgs t;
      if (int st = fill_tc(cs[r], L, a, boff, mode, dvk, sent, M, chunks_b, t, chunks, os[r])) return st;
      if (r == 0) t0 = t;
      if (S > 1) {
        t0.Ur[r] = t.U;
        for (int q = 0; q < nef::kMaxTabs; ++q) t0.tabr[r][q] = t.tab[q];
        t0.Qpartr[r] = t.Qpart;
        t0.losspartr[r] = t.losspart;
        t0.countpartr[r] = t.countpart;
        t0.vdr[r] = t.vd_rows_ptr;
      }
    }
    t0.nrs = S > 1 ? S : 0;
    prof_begin(c.s);
    CK(nef::tc::launch(t0, Yk, Mk, L.tc_row_blocks, chunks, c.s, c.aux));
    prof_end(c.s, bytes);
    ++g_launches;
    return NEF_OK;
  }
  for (int r = 0; r < S; ++r) {
    nef::FusedArgs a = fused_args(cs[r], L, Y, M, mode, dv, boff);
    prof_begin(c.s);
    CK(nef::launch_fused_ffma(a, c.s));
    prof_end(c.s, bytes);
    ++g_launches;
    StreamOut& o = os[r];
    o.Qpart = a.Qpart;
    o.n_chunks = L.n_chunks;
    o.losspart = a.losspart;
    o.countpart = a.countpart;
    o.nparts = ((L.n_rows + 63) / 64) * L.n_chunks;
  }
  return NEF_OK;
}

int stream_pass(const Ctx& c, const nef::Lowering& L, const float* Y, const uint8_t* M, int mode,
                const nef::DivParams& dv, StreamOut& o) {
  return stream_pass_multi(&c, 1, L, Y, M, mode, dv, &o);
}

bool communicates(const nef::Plan& p);
int allreduce(const nef::Plan& p, void* buf, size_t count, int dtype, cudaStream_t s);

// Loss partials of one pass -> slot[r] (double) + cslot[r] (long long), one role (three on a split
// fit); then, for split fits, the slots go to pinned host memory behind an event (Ctx::pin)
int reduce_loss(const Ctx& c, const StreamOut& o, const uint8_t* M, double* slot, long long* cslot) {
  const int nrole = (c.split && M) ? 3 : 1;
  for (int q = 0; q < nrole; ++q) {
    CK(nef::launch_loss_reduce(o.losspart + q * o.nparts, o.countpart + q * o.nparts, o.nparts, slot + q, cslot + q,
                               c.s, o.lconst ? c.lscale : 1.0, o.lconst ? c.loff : nullptr));
    ++g_launches;
  }
  if (c.pin) {
    if (communicates(*c.p)) {
      if (int r = allreduce(*c.p, slot, 3, kNcclFloat64, c.s)) return r;
      if (c.pin_counts)
        if (int r = allreduce(*c.p, cslot, 3, kNcclInt64, c.s)) return r;
    }
    CK(cudaMemcpyAsync(c.pin, slot, 3 * sizeof(double), cudaMemcpyDeviceToHost, c.s));
    if (c.pin_counts) CK(cudaMemcpyAsync(static_cast<char*>(c.pin) + 32, cslot, 3 * sizeof(long long), cudaMemcpyDeviceToHost, c.s));
    CK(cudaEventRecord(c.pin_ev, c.s));
  }
  return NEF_OK;
}

// Loss-only pass with lowering 0 -> slot (double) + count slot (long long)
int loss_pass(const Ctx& c, const float* Y, const uint8_t* M, const nef::DivParams& dv, double* slot, long long* cslot) {
  const nef::Lowering& L = c.p->low[0];
  int st = side_operands(c, L);
  if (st) return st;
  StreamOut o;
  if ((st = stream_pass(c, L, Y, M, 2, dv, o))) return st;
  return reduce_loss(c, o, M, slot, cslot);
}

// Steps 1-4 of one factor update: leaves A in *num, B in *den (device pointers into ws).  With
// `fused` (epilogue-free lowering, no all-reduce) the split partials are left unreduced in *fused
// for the fused reduce + update kernel and num / den are not written.
// After the streamed pass of factor ell: the loss slots (mode 1), then A | B - the split
// partials reduced in fixed order and the epilogue einsum (einstr_ell on the row side) - left in
// *num / *den.  With `fused` (epilogue-free lowering, no all-reduce) the partials stay unreduced
// for the fused reduce + update kernel and num / den are not written.
int finish_num_den(const Ctx& c, int ell, const uint8_t* M, int mode, double* slot, long long* cslot,
                   const StreamOut& o, float** num, float** den, bool fused) {
  const nef::Lowering& L = c.p->low[ell];
  int st;
  if (mode == 1 && (st = reduce_loss(c, o, M, slot, cslot))) return st;
  if (fused && L.epi_identity) return NEF_OK;
  const int64_t qe = L.n_rows * L.K;
  float* Q = reinterpret_cast<float*>(c.ws + L.ws_Q);
  CK(nef::launch_reduce_q(o.Qpart, Q, o.n_chunks, 2 * qe, c.s));
  ++g_launches;
  if (L.epi_identity) {
    *num = Q;
    *den = Q + qe;
    return NEF_OK;
  }
  st = run_prog(c, L.epi);                                            // A from Q_a
  if (st) return st;
  st = run_prog(c, L.epi, L.ws_Q, L.ws_Q + qe * 4, L.ws_num, L.ws_den);  // B from Q_b
  if (st) return st;
  *num = reinterpret_cast<float*>(c.ws + L.ws_num);
  *den = reinterpret_cast<float*>(c.ws + L.ws_den);
  return NEF_OK;
}

// Steps 1-4 of one factor update: leaves A in *num, B in *den (device pointers into ws).
int num_den(const Ctx& c, int ell, const float* Y, const uint8_t* M, const nef::DivParams& dv, int mode,
            double* slot, long long* cslot, float** num, float** den) {
  const nef::Lowering& L = c.p->low[ell];
  int st = side_operands(c, L);
  if (st) return st;
  StreamOut o;
  if ((st = stream_pass(c, L, Y, M, mode, dv, o))) return st;
  return finish_num_den(c, ell, M, mode, slot, cslot, o, num, den, false);
}

// A plan "communicates" when it is sharded over > 1 ranks, or carries a 1-rank communicator
// (NEF_NCCL_FORCE=1 at nef_plan_shard with world 1: the multi-GPU code path, NCCL included,
// exercised on one GPU by the tests)
bool communicates(const nef::Plan& p) { return p.world > 1 || p.nccl_comm != nullptr; }

int allreduce(const nef::Plan& p, void* buf, size_t count, int dtype, cudaStream_t s) {
  if (!communicates(p)) return NEF_OK;
  if (!p.nccl_comm)
    return fail(NEF_E_NCCL, "plan sharded without a communicator (nef_plan_shard_host): use nef_num_den, an "
                            "external all-reduce and nef_apply_update");
  int r = g_nccl.AllReduce(buf, buf, count, dtype, kNcclSum, p.nccl_comm, s);
  if (r != 0) return fail(NEF_E_NCCL, std::string("ncclAllReduce: ") + (g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?"));
  return NEF_OK;
}

// Steps 5-6 after the streamed pass: finish A | B, all-reduce (sharded plans, factors without the
// shard mode), update.  Epilogue-free lowerings on one rank reduce and update in one launch.
int finish_update(const Ctx& c, int ell, const uint8_t* M, const nef::UpdArgs& u, int mode, double* slot,
                  long long* cslot, const StreamOut& o) {
  int64_t n = 1;
  for (auto d : c.p->fshape[ell]) n *= d;
  const bool fuse = !communicates(*c.p) && c.p->low[ell].epi_identity;
  float *num = nullptr, *den = nullptr;
  int st = finish_num_den(c, ell, M, mode, slot, cslot, o, &num, &den, fuse);
  if (st) return st;
  if (fuse) {   // numerator / denominator summed from the split partials inside the update kernel
    CK(nef::launch_reduce_update(o.Qpart, c.F[ell], o.n_chunks, n, u, c.s));
    ++g_launches;
    return NEF_OK;
  }
  if (communicates(*c.p) && !c.p->factor_has_shard[ell]) {
    // num and den are adjacent in the workspace (Q_a|Q_b or num|den regions)
    if (den == num + n) {
      st = allreduce(*c.p, num, 2 * (size_t)n, kNcclFloat32, c.s);
    } else {
      st = allreduce(*c.p, num, (size_t)n, kNcclFloat32, c.s);
      if (!st) st = allreduce(*c.p, den, (size_t)n, kNcclFloat32, c.s);
    }
    if (st) return st;
  }
  CK(nef::launch_update(c.F[ell], num, den, n, u, c.s));
  ++g_launches;
  return NEF_OK;
}

int update_one(const Ctx& c, int ell, const float* Y, const uint8_t* M, const nef::DivParams& dv, const nef::UpdArgs& u,
               int mode, double* slot, long long* cslot) {
  const nef::Lowering& L = c.p->low[ell];
  int st = side_operands(c, L);
  if (st) return st;
  StreamOut o;
  if ((st = stream_pass(c, L, Y, M, mode, dv, o))) return st;
  return finish_update(c, ell, M, u, mode, slot, cslot, o);
}

int validate_ab(double alpha, double beta) {
  if (!std::isfinite(alpha) || !std::isfinite(beta)) return fail(NEF_E_DOMAIN, "non-finite alpha/beta");
  if (alpha == 0.0 && beta != 1.0)
    return fail(NEF_E_DOMAIN, "alpha = 0 requires beta = 1: no decomposition satisfying eq:prop (P:529)");
  return NEF_OK;
}

int validate_common(nef_plan_t plan, const float* Y, float* const* factors, void* ws, size_t ws_bytes) {
  if (!plan) return fail(NEF_E_ARG, "null plan");
  if (!Y || (reinterpret_cast<uintptr_t>(Y) & 15)) return fail(NEF_E_ARG, "Y must be a non-null 16-byte aligned device pointer");
  if (!factors) return fail(NEF_E_ARG, "null factor array");
  for (size_t l = 0; l < plan->p.ops.size(); ++l)
    if (!factors[l] || (reinterpret_cast<uintptr_t>(factors[l]) & 3)) return fail(NEF_E_ARG, "null or misaligned factor pointer");
  if (!ws || ws_bytes < plan->p.ws_bytes)
    return fail(NEF_E_ARG, "workspace too small: need " + std::to_string(plan->p.ws_bytes) + " bytes");
  if (reinterpret_cast<uintptr_t>(ws) & 255) return fail(NEF_E_ARG, "workspace must be 256-byte aligned");
  return NEF_OK;
}

// loss specification (include/nef.h nef_loss_spec), validated
struct Spec {
  int fam = nef::FAM_AB;
  double alpha = 1.0, beta = 0.0, prm = 0.0;
  const float* aux = nullptr;
};

nef_loss_spec ab_spec(double alpha, double beta) {
  nef_loss_spec l{};
  l.kind = NEF_LOSS_AB;
  l.alpha = alpha;
  l.beta = beta;
  return l;
}

int validate_spec(const nef_loss_spec* l, Spec& sp) {
  if (!l) return fail(NEF_E_ARG, "null loss spec");
  if (l->kind < NEF_LOSS_AB || l->kind > NEF_LOSS_JS) return fail(NEF_E_DOMAIN, "unknown loss kind");
  sp.fam = l->kind;
  if (l->kind == NEF_LOSS_AB) {
    if (int st = validate_ab(l->alpha, l->beta)) return st;
    sp.alpha = l->alpha;
    sp.beta = l->beta;
  }
  if (l->kind == NEF_LOSS_NEGBIN || l->kind == NEF_LOSS_BINOMIAL) {
    if (l->aux) {
      if (reinterpret_cast<uintptr_t>(l->aux) & 3) return fail(NEF_E_ARG, "misaligned aux tensor");
      sp.aux = l->aux;
    } else if (!(l->param > 0.0) || !std::isfinite(l->param)) {
      return fail(NEF_E_DOMAIN, l->kind == NEF_LOSS_NEGBIN ? "negative binomial needs phi > 0 (P:543)"
                                                           : "binomial needs n > 0 trials (P:587)");
    }
    sp.prm = l->param;
  } else if (l->aux) {
    return fail(NEF_E_ARG, "aux tensor given for a loss without per-entry parameters");
  }
  return NEF_OK;
}

// ------------------------------------------------------------------ sweep graphs
// One sweep of nef_fit captured as a CUDA graph (cached per plan for one input set): the loss of
// the iterate entering the sweep goes to a fixed slot and a one-thread kernel appends it to the
// trace at a device-side counter, so the graph is identical for every sweep.  The streaming
// launches keep their CUDA-event timing as external event-record nodes, re-pointed at fresh
// profiling events before each replay when nef_profile is on.
std::string sweep_key(const Ctx& c, const float* Y, const uint8_t* M, const nef::DivParams& dv, const nef::UpdArgs& u) {
  std::string k;
  char buf[128];
  auto add = [&](const void* q) { std::snprintf(buf, sizeof buf, "%p,", q); k += buf; };
  add(Y); add(M); add(c.ws); add(c.ysent); add(c.loff); add(c.aux);
  for (size_t l = 0; l < c.p->ops.size(); ++l) add(c.F[l]);
  std::snprintf(buf, sizeof buf, "%zu,%d,%d,%d,%.17g,%d,", c.ws_bytes, g_policy, (int)g_vdirect, (int)c.sqy, c.lscale,
                (int)g_no_memo);
  k += buf;
  k.append(reinterpret_cast<const char*>(&dv), sizeof dv);
  k.append(reinterpret_cast<const char*>(&u), sizeof u);
  return k;
}

int update_one(const Ctx& c, int ell, const float* Y, const uint8_t* M, const nef::DivParams& dv, const nef::UpdArgs& u,
               int mode, double* slot, long long* cslot);

SweepGraph* sweep_graph(nef_plan_t plan, const Ctx& c, const float* Y, const uint8_t* M, const nef::DivParams& dv,
                        const nef::UpdArgs& u, double* slots, long long* cslots) {
  const std::string key = sweep_key(c, Y, M, dv, u);
  if (plan->g && plan->g->key == key) return plan->g;
  if (plan->graph_failed) return nullptr;
  delete plan->g;
  plan->g = nullptr;
  if (!plan->cap_stream && cudaStreamCreateWithFlags(&plan->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    plan->graph_failed = true;
    return nullptr;
  }
  Ctx cc = c;                 // captured on the private stream; replayed on the caller's
  cc.s = plan->cap_stream;
  cc.memo = !g_no_memo;       // the updates run in order 0, 1, ... below
  auto* sg = new SweepGraph();
  sg->key = key;
  const int kSlots = 2048;
  double* fixed = slots + kSlots - 2;
  long long* cfixed = cslots + kSlots - 2;
  long long* ctr = cslots + kSlots - 1;
  const int64_t launches0 = g_launches;
  const std::string err0 = g_err;
  if (cudaStreamBeginCapture(cc.s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    plan->graph_failed = true;
    delete sg;
    return nullptr;
  }
  g_prof.cap = sg;
  int st = NEF_OK;
  for (int ell = 0; ell < (int)c.p->ops.size() && !st; ++ell)
    st = update_one(cc, ell, Y, M, dv, u, ell == 0 ? 1 : 0, fixed, cfixed);
  if (!st && nef::launch_slot_push(fixed, cfixed, slots, cslots, ctr, cc.s) != cudaSuccess) st = NEF_E_CUDA;
  g_prof.cap = nullptr;
  cudaGraph_t graph = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(cc.s, &graph);
  g_launches = launches0;
  if (st || ec != cudaSuccess || !graph) {   // fall back to plain launches for this plan
    if (graph) cudaGraphDestroy(graph);
    cudaGetLastError();
    g_err = err0;
    plan->graph_failed = true;
    delete sg;
    return nullptr;
  }
  sg->graph = graph;
  if (cudaGraphInstantiate(&sg->exec, graph, 0) != cudaSuccess) {
    cudaGetLastError();
    plan->graph_failed = true;
    delete sg;
    return nullptr;
  }
  // event-record nodes in capture order (matched through their events)
  size_t nn = 0;
  cudaGraphGetNodes(graph, nullptr, &nn);
  std::vector<cudaGraphNode_t> nodes(nn);
  cudaGraphGetNodes(graph, nodes.data(), &nn);
  sg->ev_nodes.assign(sg->own.size(), nullptr);
  for (auto nd : nodes) {
    cudaGraphNodeType ty;
    cudaGraphNodeGetType(nd, &ty);
    if (ty != cudaGraphNodeTypeEventRecord) continue;
    cudaEvent_t e;
    cudaGraphEventRecordNodeGetEvent(nd, &e);
    for (size_t i = 0; i < sg->own.size(); ++i)
      if (sg->own[i] == e) sg->ev_nodes[i] = nd;
  }
  for (auto nd : sg->ev_nodes)
    if (!nd) { delete sg; return nullptr; }
  plan->g = sg;
  return sg;
}

int replay_sweep(SweepGraph* sg, cudaStream_t s) {
  const size_t nl = sg->bytes.size();   // streaming launches per sweep
  if (g_prof.on) {
    for (size_t i = 0; i < nl; ++i) {
      if (!prof_reserve()) break;
      cudaGraphExecEventRecordNodeSetEvent(sg->exec, sg->ev_nodes[2 * i], g_prof.ev[2 * g_prof.used]);
      cudaGraphExecEventRecordNodeSetEvent(sg->exec, sg->ev_nodes[2 * i + 1], g_prof.ev[2 * g_prof.used + 1]);
      g_prof.used++;
      g_prof.bytes += sg->bytes[i];
    }
    sg->on_prof = true;
  } else if (sg->on_prof) {
    for (size_t i = 0; i < sg->own.size(); ++i) cudaGraphExecEventRecordNodeSetEvent(sg->exec, sg->ev_nodes[i], sg->own[i]);
    sg->on_prof = false;
  }
  CK(cudaGraphLaunch(sg->exec, s));
  size_t n = 0;
  cudaGraphGetNodes(sg->graph, nullptr, &n);
  g_launches += (int64_t)(n - sg->own.size());   // kernel (and push) nodes of the sweep
  return NEF_OK;
}

int check_device() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(NEF_E_CUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
  return NEF_OK;
}

}  // namespace

extern "C" {

const char* nef_last_error(void) { return g_err.c_str(); }
const char* nef_version(void) { return "nef 0.1 (sm_100a)"; }
int64_t nef_last_launch_count(void) { return g_launches; }
int nef_profile_enable(int enable) {
  g_prof.on = enable != 0;
  g_prof.used = 0;
  g_prof.bytes = 0;
  return NEF_OK;
}

int nef_profile_read(double* kernel_ms, int64_t* launches, double* algorithmic_bytes) {
  double ms = 0;
  if (g_prof.used) {
    cudaError_t e = cudaEventSynchronize(g_prof.ev[2 * g_prof.used - 1]);
    if (e != cudaSuccess) return fail(NEF_E_CUDA, std::string("cudaEventSynchronize: ") + cudaGetErrorString(e));
    for (size_t i = 0; i < g_prof.used; ++i) {
      float t = 0;
      e = cudaEventElapsedTime(&t, g_prof.ev[2 * i], g_prof.ev[2 * i + 1]);
      if (e != cudaSuccess) return fail(NEF_E_CUDA, std::string("cudaEventElapsedTime: ") + cudaGetErrorString(e));
      ms += t;
    }
  }
  if (kernel_ms) *kernel_ms = ms;
  if (launches) *launches = (int64_t)g_prof.used;
  if (algorithmic_bytes) *algorithmic_bytes = g_prof.bytes;
  return NEF_OK;
}

int nef_debug_dump(float* device_buffer) {
  g_debug = device_buffer;
  return NEF_OK;
}

int nef_debug_trace(int64_t* device_buffer) {
  g_trace = reinterpret_cast<long long*>(device_buffer);
  return NEF_OK;
}

int nef_set_kernel_policy(int policy) {
  if (policy < 0 || policy > 7) return fail(NEF_E_ARG, "policy must be 0..7");
  g_policy = policy & 1;
  g_graphs = (policy & 2) == 0 && [] { const char* e = std::getenv("NEF_NO_GRAPH"); return !e || e[0] != '1'; }();
  g_no_memo = (policy & 4) != 0 || std::getenv("NEF_NO_REUSE") != nullptr;
  return NEF_OK;
}

int nef_plan(const char* einsum, int n_modes, const int64_t* shape, int n_ranks, const int64_t* ranks, nef_plan_t* out) {
  if (!out) return fail(NEF_E_ARG, "null out");
  *out = nullptr;
  auto* h = new nef_plan_s();
  std::string err;
  int st = nef::build_plan(einsum, n_modes, shape, n_ranks, ranks, h->p, err);
  if (st) {
    delete h;
    return fail(st, err);
  }
  *out = h;
  return NEF_OK;
}

void nef_plan_destroy(nef_plan_t plan) {
  if (!plan) return;
  if (plan->p.nccl_comm && g_nccl.loaded) g_nccl.CommDestroy(plan->p.nccl_comm);
  delete plan;
}

int nef_plan_info(nef_plan_t plan, int* n_factors, int* shard_mode, int64_t* local_begin, int64_t* local_len,
                  size_t* workspace_bytes) {
  if (!plan) return fail(NEF_E_ARG, "null plan");
  if (n_factors) *n_factors = (int)plan->p.ops.size();
  if (shard_mode) *shard_mode = plan->p.shard_mode;
  if (local_begin) *local_begin = plan->p.local_begin;
  if (local_len) *local_len = plan->p.local_len;
  if (workspace_bytes) *workspace_bytes = plan->p.ws_bytes;
  return NEF_OK;
}

int nef_factor_shape(nef_plan_t plan, int ell, int64_t* dims, int* ndim) {
  if (!plan || !dims || !ndim) return fail(NEF_E_ARG, "null argument");
  if (ell < 0 || ell >= (int)plan->p.ops.size()) return fail(NEF_E_ARG, "ell out of range");
  const auto& s = plan->p.fshape[ell];
  *ndim = (int)s.size();
  for (size_t k = 0; k < s.size(); ++k) dims[k] = s[k];
  return NEF_OK;
}

int nef_local_shape(nef_plan_t plan, int64_t* dims, int* ndim) {
  if (!plan || !dims || !ndim) return fail(NEF_E_ARG, "null argument");
  *ndim = (int)plan->p.shape.size();
  for (size_t k = 0; k < plan->p.shape.size(); ++k) dims[k] = plan->p.shape[k];
  return NEF_OK;
}

int nef_plan_describe(nef_plan_t plan, char* buf, size_t cap, size_t* len) {
  if (!plan) return fail(NEF_E_ARG, "null plan");
  std::string s = nef::describe_plan(plan->p);
  if (len) *len = s.size() + 1;
  if (buf && cap) {
    size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return NEF_OK;
}

int nef_fit_ex(nef_plan_t plan, const float* Y, const uint8_t* mask, const nef_loss_spec* loss, double eps,
               float* const* factors, int iters, double* loss_trace, void* workspace, size_t ws_bytes, void* stream) {
  int st = validate_common(plan, Y, factors, workspace, ws_bytes);
  if (st) return st;
  Spec sp;
  if ((st = validate_spec(loss, sp))) return st;
  if (!(eps > 0.0) || !std::isfinite(eps)) return fail(NEF_E_ARG, "eps must be > 0");
  if (iters < 0) return fail(NEF_E_ARG, "iters must be >= 0");
  if (int dst = check_device()) return dst;
  g_launches = 0;
  const nef::Plan& p = plan->p;
  Ctx c{&p, factors, static_cast<char*>(workspace), ws_bytes, static_cast<cudaStream_t>(stream)};
  c.aux = sp.aux;
  nef::DivParams dv = nef::make_div_fam(sp.fam, sp.alpha, sp.beta, sp.prm);
  nef::UpdArgs u = nef::make_upd_fam(sp.fam, sp.alpha, sp.beta, eps);
  // a1 precompute (once per fit): fold the mask into a NaN-sentinel copy of Y for the tcgen05
  // passes (R5: missing values are never used, whatever Y holds there)
  // R25: for the pairs that split the loss, its data-only part is summed once per fit (with the
  // sentinel copy when there is a mask, else by a read-only pass) when the loss-carrying
  // lowering runs on the tcgen05 kernel
  const int dterm = (g_no_lconst || g_policy != 0 || sp.fam != nef::FAM_AB) ? 0
                    : dv.kind == nef::EW_B_M05   ? 1
                    : dv.kind == nef::EW_KL      ? 2
                    : dv.kind == nef::EW_A05_B0  ? 3
                                                 : 0;
  const double lscale = dterm == 1 ? 2.0 : dterm == 3 ? 4.0 : 1.0;
  double* dslot = reinterpret_cast<double*>(c.ws + p.ws_dterm);
  double* dpart = reinterpret_cast<double*>(c.ws + p.ws_dpart);
  long long* dcpart = reinterpret_cast<long long*>(dpart + nef::kSentParts);
  bool any_tc = false;
  for (const auto& L : p.low) any_tc |= L.tc_ok;
  // R35: the (0.5, 0) pair needs the data only as sqrt(y) (a = y^(1/2) yhat^-1, the loss split of
  // R25): the once-per-fit copy holds sqrt(y), masked or not, and the passes save one MUFU per entry
  c.sqy = dv.kind == nef::EW_A05_B0 && any_tc && g_policy == 0 && !g_no_sentinel && !sp.aux && !g_no_sqy;
  if ((mask || c.sqy) && g_policy == 0 && !g_no_sentinel) {
    if (any_tc) {
      float* ys = reinterpret_cast<float*>(c.ws + p.ws_sent);
      CK(nef::launch_sentinel(Y, mask, ys, p.n_local, dterm, dpart, dcpart, dslot,
                              reinterpret_cast<long long*>(dslot + 1), c.s, 0, c.sqy ? 1 : 0));
      g_launches += 3;
      c.ysent = ys;
      if (dterm) {
        c.loff = dslot;
        c.lscale = lscale;
      }
    }
  } else if (!mask && dterm && p.low[0].tc_ok && iters >= 3 && !sp.aux) {
    // (the read-only pass costs about what the split saves on two loss-carrying passes)
    CK(nef::launch_dterm(Y, p.n_local, dterm, dpart, dcpart, dslot, reinterpret_cast<long long*>(dslot + 1), c.s));
    g_launches += 3;
    c.loff = dslot;
    c.lscale = lscale;
  }
  double* slots = reinterpret_cast<double*>(c.ws + p.ws_trace);
  long long* cslots = reinterpret_cast<long long*>(c.ws + p.ws_trace + 8 * 2048);
  const int kSlots = 2048;
  std::vector<double> host(iters + 1);
  int base = 0;   // trace index of slot 0
  auto flush = [&](int upto) -> int {
    // all-reduce the loss slots [0, upto - base) and copy them to the host
    int n = upto - base;
    if (n <= 0) return NEF_OK;
    if (communicates(p)) {
      int r = allreduce(p, slots, (size_t)n, kNcclFloat64, c.s);
      if (r) return r;
    }
    CK(cudaMemcpyAsync(host.data() + base, slots, sizeof(double) * n, cudaMemcpyDeviceToHost, c.s));
    CK(cudaStreamSynchronize(c.s));
    base = upto;
    return NEF_OK;
  };
  // Sweeps: replay a captured one-sweep CUDA graph (launch-bound small problems: one submission
  // per sweep instead of ~25) when the plan runs on one rank and the trace fits the slots; else
  // launch the sweep's kernels one by one.
  int t0 = 0;
  if (g_graphs && !communicates(p) && iters >= 2 && iters + 1 <= kSlots - 2) {
    SweepGraph* sg = sweep_graph(plan, c, Y, mask, dv, u, slots, cslots);
    if (sg) {
      CK(cudaMemsetAsync(cslots + kSlots - 1, 0, sizeof(long long), c.s));   // slot counter
      for (int t = 0; t < iters; ++t)
        if ((st = replay_sweep(sg, c.s))) return st;
      t0 = iters;
    }
  }
  Ctx cm = c;
  cm.memo = !g_no_memo;   // one sweep = the updates in order 0, 1, ...
  for (int t = t0; t < iters; ++t) {
    if (t - base >= kSlots) { if ((st = flush(t))) return st; }
    for (int ell = 0; ell < (int)p.ops.size(); ++ell) {
      int mode = (ell == 0) ? 1 : 0;
      st = update_one(cm, ell, Y, mask, dv, u, mode, slots + (t - base), cslots + (t - base));
      if (st) return st;
    }
  }
  if (iters - base >= kSlots) { if ((st = flush(iters))) return st; }
  st = loss_pass(c, Y, mask, dv, slots + (iters - base), cslots + (iters - base));
  if (st) return st;
  if ((st = flush(iters + 1))) return st;
  if (loss_trace) std::memcpy(loss_trace, host.data(), sizeof(double) * (iters + 1));
  return NEF_OK;
}

int nef_fit(nef_plan_t plan, const float* Y, const uint8_t* mask, double alpha, double beta, double eps,
            float* const* factors, int iters, double* loss_trace, void* workspace, size_t ws_bytes, void* stream) {
  const nef_loss_spec ls = ab_spec(alpha, beta);
  return nef_fit_ex(plan, Y, mask, &ls, eps, factors, iters, loss_trace, workspace, ws_bytes, stream);
}

// Batched random restarts (N4): S independent fits of the same data, each factor
// update's streamed pass launched ONCE for all restarts (grid z = restart) so that the restarts'
// CTAs read the same Y tiles together - one HBM stream, the other restarts served by L2.
size_t nef_restarts_workspace_bytes(nef_plan_t plan, int restarts) {
  if (!plan || restarts < 1) return 0;
  const nef::Plan& p = plan->p;
  const size_t per = ((size_t)p.ws_sent + 255) / 256 * 256;   // everything but the sentinel copy
  return per * (size_t)restarts + (size_t)p.n_local * 4 + 256;
}

int nef_fit_restarts(nef_plan_t plan, const float* Y, const uint8_t* mask, const nef_loss_spec* loss, double eps,
                     float* const* factors, int restarts, int iters, double* loss_traces, void* workspace,
                     size_t ws_bytes, void* stream) {
  if (!plan) return fail(NEF_E_ARG, "null plan");
  const nef::Plan& p = plan->p;
  const int S = restarts;
  if (S < 1) return fail(NEF_E_ARG, "restarts must be >= 1");
  if (iters < 0 || iters >= 2048) return fail(NEF_E_ARG, "iters must be in [0, 2048) for batched restarts");
  if (!Y || (reinterpret_cast<uintptr_t>(Y) & 15)) return fail(NEF_E_ARG, "Y must be a non-null 16-byte aligned device pointer");
  if (!factors) return fail(NEF_E_ARG, "null factor array");
  const int L = (int)p.ops.size();
  for (int i = 0; i < S * L; ++i)
    if (!factors[i] || (reinterpret_cast<uintptr_t>(factors[i]) & 3)) return fail(NEF_E_ARG, "null or misaligned factor pointer");
  if (!workspace || ws_bytes < nef_restarts_workspace_bytes(plan, S))
    return fail(NEF_E_ARG, "workspace too small: need " + std::to_string(nef_restarts_workspace_bytes(plan, S)) + " bytes");
  if (reinterpret_cast<uintptr_t>(workspace) & 255) return fail(NEF_E_ARG, "workspace must be 256-byte aligned");
  Spec sp;
  int st = validate_spec(loss, sp);
  if (st) return st;
  if (!(eps > 0.0) || !std::isfinite(eps)) return fail(NEF_E_ARG, "eps must be > 0");
  if (int dst = check_device()) return dst;
  g_launches = 0;
  const size_t per = ((size_t)p.ws_sent + 255) / 256 * 256;
  char* ws = static_cast<char*>(workspace);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<Ctx> cs(S);
  for (int r = 0; r < S; ++r) {
    cs[r] = Ctx{&p, factors + (size_t)r * L, ws + r * per, per, s};
    cs[r].aux = sp.aux;
  }
  const nef::DivParams dv = nef::make_div_fam(sp.fam, sp.alpha, sp.beta, sp.prm);
  const nef::UpdArgs u = nef::make_upd_fam(sp.fam, sp.alpha, sp.beta, eps);
  // once per fit, shared by the restarts: the sentinel copy (and its data-only loss sum, R25)
  const int dterm = (g_no_lconst || g_policy != 0 || sp.fam != nef::FAM_AB) ? 0
                    : dv.kind == nef::EW_B_M05   ? 1
                    : dv.kind == nef::EW_KL      ? 2
                    : dv.kind == nef::EW_A05_B0  ? 3
                                                 : 0;
  bool any_tc = false;
  for (const auto& Lw : p.low) any_tc |= Lw.tc_ok;
  const bool sqy = dv.kind == nef::EW_A05_B0 && any_tc && g_policy == 0 && !g_no_sentinel && !sp.aux && !g_no_sqy;
  if ((mask || sqy) && any_tc && g_policy == 0 && !g_no_sentinel) {
    double* dslot = reinterpret_cast<double*>(ws + p.ws_dterm);
    double* dpart = reinterpret_cast<double*>(ws + p.ws_dpart);
    float* ys = reinterpret_cast<float*>(ws + per * S);
    CK(nef::launch_sentinel(Y, mask, ys, p.n_local, dterm, dpart, reinterpret_cast<long long*>(dpart + nef::kSentParts),
                            dslot, reinterpret_cast<long long*>(dslot + 1), s, 0, sqy ? 1 : 0));
    g_launches += 3;
    for (auto& c : cs) {
      c.ysent = ys;
      c.sqy = sqy;
      if (dterm) {
        c.loff = dslot;
        c.lscale = dterm == 1 ? 2.0 : dterm == 3 ? 4.0 : 1.0;
      }
    }
  }
  std::vector<StreamOut> os(S);
  auto slot = [&](int r) { return reinterpret_cast<double*>(cs[r].ws + p.ws_trace); };
  auto cslot = [&](int r) { return reinterpret_cast<long long*>(cs[r].ws + p.ws_trace + 8 * 2048); };
  for (int t = 0; t <= iters; ++t) {
    const bool last = t == iters;   // the final loss-only pass
    for (int ell = 0; ell < (last ? 1 : L); ++ell) {
      const nef::Lowering& Lw = p.low[ell];
      const int mode = last ? 2 : (ell == 0 ? 1 : 0);
      for (int r = 0; r < S; ++r)
        if ((st = side_operands(cs[r], Lw))) return st;
      if ((st = stream_pass_multi(cs.data(), S, Lw, Y, mask, mode, dv, os.data()))) return st;
      for (int r = 0; r < S; ++r) {
        if (last) st = reduce_loss(cs[r], os[r], mask, slot(r) + t, cslot(r) + t);
        else st = finish_update(cs[r], ell, mask, u, mode, slot(r) + t, cslot(r) + t, os[r]);
        if (st) return st;
      }
    }
  }
  std::vector<double> host((size_t)S * (iters + 1));
  for (int r = 0; r < S; ++r) {
    if (communicates(p))
      if ((st = allreduce(p, slot(r), (size_t)iters + 1, kNcclFloat64, s))) return st;
    CK(cudaMemcpyAsync(host.data() + (size_t)r * (iters + 1), slot(r), sizeof(double) * (iters + 1),
                       cudaMemcpyDeviceToHost, s));
  }
  CK(cudaStreamSynchronize(s));
  if (loss_traces) std::memcpy(loss_traces, host.data(), sizeof(double) * host.size());
  return NEF_OK;
}

// Train / validation / heldout fit with the stopping rules of P:497 (readings R29-R32).  Per
// sweep t + 1, the first factor's pass also yields the three loss sums of the iterate t that
// enters it; they reach pinned host memory behind an event while the rest of the sweep runs, the
// host applies the rules, and on a stop the factors saved before sweep t + 1 (iterate t) are
// restored.
int nef_fit_split(nef_plan_t plan, const float* Y, const uint8_t* labels, const nef_loss_spec* loss, double eps,
                  float* const* factors, const nef_stop_rule* rule, double* traces, int64_t* counts, int* sweeps,
                  int* reason, void* workspace, size_t ws_bytes, void* stream) {
  int st = validate_common(plan, Y, factors, workspace, ws_bytes);
  if (st) return st;
  Spec sp;
  if ((st = validate_spec(loss, sp))) return st;
  if (!labels) return fail(NEF_E_ARG, "null labels");
  if (!rule || rule->max_iters < 0 || rule->val_patience < 0 || !(rule->min_rel_decrease == rule->min_rel_decrease))
    return fail(NEF_E_ARG, "bad stop rule");
  if (!(eps > 0.0) || !std::isfinite(eps)) return fail(NEF_E_ARG, "eps must be > 0");
  if (int dst = check_device()) return dst;
  g_launches = 0;
  const nef::Plan& p = plan->p;
  Ctx c{&p, factors, static_cast<char*>(workspace), ws_bytes, static_cast<cudaStream_t>(stream)};
  c.aux = sp.aux;
  c.split = 1;
  const nef::DivParams dv = nef::make_div_fam(sp.fam, sp.alpha, sp.beta, sp.prm);
  const nef::UpdArgs u = nef::make_upd_fam(sp.fam, sp.alpha, sp.beta, eps);
  bool any_tc = false;
  for (const auto& L : p.low) any_tc |= L.tc_ok;
  if (any_tc && g_policy == 0 && !g_no_sentinel) {   // train entries folded into a sentinel copy
    double* dslot = reinterpret_cast<double*>(c.ws + p.ws_dterm);
    double* dpart = reinterpret_cast<double*>(c.ws + p.ws_dpart);
    float* ys = reinterpret_cast<float*>(c.ws + p.ws_sent);
    CK(nef::launch_sentinel(Y, labels, ys, p.n_local, 0, dpart, reinterpret_cast<long long*>(dpart + nef::kSentParts),
                            dslot, reinterpret_cast<long long*>(dslot + 1), c.s, 1));
    g_launches += 3;
    c.ysent = ys;
  }
  const int L = (int)p.ops.size();
  std::vector<float*> fsave(L);
  std::vector<size_t> fbytes(L);
  {
    char* q = c.ws + p.ws_fsave;
    for (int l = 0; l < L; ++l) {
      size_t n = 1;
      for (auto d : p.fshape[l]) n *= (size_t)d;
      fbytes[l] = n * 4;
      fsave[l] = reinterpret_cast<float*>(q);
      q += (n * 4 + 255) / 256 * 256;
    }
  }
  void* pin = nullptr;
  CK(cudaHostAlloc(&pin, 64, cudaHostAllocDefault));
  cudaEvent_t ev = nullptr;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess) {
    cudaFreeHost(pin);
    return fail(NEF_E_CUDA, "cudaEventCreate failed");
  }
  c.pin = pin;
  c.pin_ev = ev;
  double* slots = reinterpret_cast<double*>(c.ws + p.ws_trace);
  long long* cslots = reinterpret_cast<long long*>(c.ws + p.ws_trace + 8 * 2048);
  const int T = rule->max_iters;
  std::vector<double> tr[3];
  int why = 0, t = 0;
  auto run = [&]() -> int {
    for (t = 0;; ++t) {
      c.pin_counts = (t == 0);
      if (t < T) {   // sweep t + 1; its first pass carries the losses of iterate t
        for (int l = 0; l < L; ++l) CK(cudaMemcpyAsync(fsave[l], factors[l], fbytes[l], cudaMemcpyDeviceToDevice, c.s));
        Ctx cm = c;
        cm.memo = !g_no_memo;   // one sweep = the updates in order 0, 1, ...
        for (int ell = 0; ell < L; ++ell)
          if (int r = update_one(cm, ell, Y, labels, dv, u, ell == 0 ? 1 : 0, slots, cslots)) return r;
      } else if (int r = loss_pass(c, Y, labels, dv, slots, cslots)) {
        return r;
      }
      CK(cudaEventSynchronize(ev));
      const double* h = static_cast<const double*>(pin);
      for (int q = 0; q < 3; ++q) tr[q].push_back(h[q]);
      if (t == 0 && counts)
        for (int q = 0; q < 3; ++q) counts[q] = static_cast<const long long*>(pin)[4 + q];
      // P:497 stopping rules (R30, R31): patience > plateau > max_iters
      const int pt = rule->val_patience;
      bool inc = pt > 0 && t >= pt;
      for (int k = t - pt + 1; inc && k <= t; ++k) inc = tr[1][k] > tr[1][k - 1];
      if (inc) why = NEF_STOP_PATIENCE;
      else if (t >= 1 && (tr[0][t - 1] - tr[0][t]) < rule->min_rel_decrease * std::fabs(tr[0][t - 1])) why = NEF_STOP_PLATEAU;
      else if (t >= T) why = NEF_STOP_MAX_ITERS;
      if (why) {
        if (t < T)   // sweep t + 1 already ran: back to iterate t
          for (int l = 0; l < L; ++l) CK(cudaMemcpyAsync(factors[l], fsave[l], fbytes[l], cudaMemcpyDeviceToDevice, c.s));
        CK(cudaStreamSynchronize(c.s));
        return NEF_OK;
      }
    }
  };
  st = run();
  cudaEventDestroy(ev);
  cudaFreeHost(pin);
  if (st) return st;
  if (traces)
    for (int q = 0; q < 3; ++q)
      for (int k = 0; k <= t; ++k) traces[(size_t)q * (T + 1) + k] = tr[q][k];
  if (sweeps) *sweeps = t;
  if (reason) *reason = why;
  return NEF_OK;
}

int nef_update_ex(nef_plan_t plan, int ell, const float* Y, const uint8_t* mask, const nef_loss_spec* loss, double eps,
                  float* const* factors, void* workspace, size_t ws_bytes, void* stream) {
  int st = validate_common(plan, Y, factors, workspace, ws_bytes);
  if (st) return st;
  Spec sp;
  if ((st = validate_spec(loss, sp))) return st;
  if (!(eps > 0.0)) return fail(NEF_E_ARG, "eps must be > 0");
  if (ell < 0 || ell >= (int)plan->p.ops.size()) return fail(NEF_E_ARG, "ell out of range");
  if (int dst = check_device()) return dst;
  g_launches = 0;
  Ctx c{&plan->p, factors, static_cast<char*>(workspace), ws_bytes, static_cast<cudaStream_t>(stream)};
  c.aux = sp.aux;
  return update_one(c, ell, Y, mask, nef::make_div_fam(sp.fam, sp.alpha, sp.beta, sp.prm),
                    nef::make_upd_fam(sp.fam, sp.alpha, sp.beta, eps), 0, nullptr, nullptr);
}

int nef_update(nef_plan_t plan, int ell, const float* Y, const uint8_t* mask, double alpha, double beta, double eps,
               float* const* factors, void* workspace, size_t ws_bytes, void* stream) {
  const nef_loss_spec ls = ab_spec(alpha, beta);
  return nef_update_ex(plan, ell, Y, mask, &ls, eps, factors, workspace, ws_bytes, stream);
}

int nef_num_den_ex(nef_plan_t plan, int ell, const float* Y, const uint8_t* mask, const nef_loss_spec* loss,
                   float* const* factors, float* num, float* den, void* workspace, size_t ws_bytes, void* stream) {
  int st = validate_common(plan, Y, factors, workspace, ws_bytes);
  if (st) return st;
  Spec sp;
  if ((st = validate_spec(loss, sp))) return st;
  if (ell < 0 || ell >= (int)plan->p.ops.size()) return fail(NEF_E_ARG, "ell out of range");
  if (!num || !den) return fail(NEF_E_ARG, "null num/den");
  if (int dst = check_device()) return dst;
  g_launches = 0;
  Ctx c{&plan->p, factors, static_cast<char*>(workspace), ws_bytes, static_cast<cudaStream_t>(stream)};
  c.aux = sp.aux;
  float *n0 = nullptr, *d0 = nullptr;
  st = num_den(c, ell, Y, mask, nef::make_div_fam(sp.fam, sp.alpha, sp.beta, sp.prm), 0, nullptr, nullptr, &n0, &d0);
  if (st) return st;
  int64_t n = 1;
  for (auto d : plan->p.fshape[ell]) n *= d;
  CK(cudaMemcpyAsync(num, n0, n * 4, cudaMemcpyDeviceToDevice, c.s));
  CK(cudaMemcpyAsync(den, d0, n * 4, cudaMemcpyDeviceToDevice, c.s));
  return NEF_OK;
}

int nef_num_den(nef_plan_t plan, int ell, const float* Y, const uint8_t* mask, double alpha, double beta,
                float* const* factors, float* num, float* den, void* workspace, size_t ws_bytes, void* stream) {
  const nef_loss_spec ls = ab_spec(alpha, beta);
  return nef_num_den_ex(plan, ell, Y, mask, &ls, factors, num, den, workspace, ws_bytes, stream);
}

int nef_apply_update_ex(nef_plan_t plan, int ell, const nef_loss_spec* loss, double eps, float* const* factors,
                        const float* num, const float* den, void* stream) {
  if (!plan || !factors || !num || !den) return fail(NEF_E_ARG, "null argument");
  Spec sp;
  int st = validate_spec(loss, sp);
  if (st) return st;
  if (ell < 0 || ell >= (int)plan->p.ops.size()) return fail(NEF_E_ARG, "ell out of range");
  if (!(eps > 0.0)) return fail(NEF_E_ARG, "eps must be > 0");
  int64_t n = 1;
  for (auto d : plan->p.fshape[ell]) n *= d;
  if (int dst = check_device()) return dst;
  g_launches = 0;
  CK(nef::launch_update(factors[ell], num, den, n, nef::make_upd_fam(sp.fam, sp.alpha, sp.beta, eps),
                        static_cast<cudaStream_t>(stream)));
  ++g_launches;
  return NEF_OK;
}

int nef_apply_update(nef_plan_t plan, int ell, double alpha, double beta, double eps, float* const* factors,
                     const float* num, const float* den, void* stream) {
  const nef_loss_spec ls = ab_spec(alpha, beta);
  return nef_apply_update_ex(plan, ell, &ls, eps, factors, num, den, stream);
}

int nef_loss_ex(nef_plan_t plan, const float* Y, const uint8_t* mask, const nef_loss_spec* loss, float* const* factors,
                double* loss_sum, int64_t* n_observed, void* workspace, size_t ws_bytes, void* stream) {
  int st = validate_common(plan, Y, factors, workspace, ws_bytes);
  if (st) return st;
  Spec sp;
  if ((st = validate_spec(loss, sp))) return st;
  if (int dst = check_device()) return dst;
  g_launches = 0;
  const nef::Plan& p = plan->p;
  Ctx c{&p, factors, static_cast<char*>(workspace), ws_bytes, static_cast<cudaStream_t>(stream)};
  c.aux = sp.aux;
  double* slot = reinterpret_cast<double*>(c.ws + p.ws_trace);
  long long* cslot = reinterpret_cast<long long*>(c.ws + p.ws_trace + 8 * 2048);
  st = loss_pass(c, Y, mask, nef::make_div_fam(sp.fam, sp.alpha, sp.beta, sp.prm), slot, cslot);
  if (st) return st;
  if (communicates(p) && p.nccl_comm) {   // (host-only split: this rank's partial sums)
    if ((st = allreduce(p, slot, 1, kNcclFloat64, c.s))) return st;
    if ((st = allreduce(p, cslot, 1, kNcclInt64, c.s))) return st;
  }
  double h = 0;
  long long hc = 0;
  CK(cudaMemcpyAsync(&h, slot, 8, cudaMemcpyDeviceToHost, c.s));
  CK(cudaMemcpyAsync(&hc, cslot, 8, cudaMemcpyDeviceToHost, c.s));
  CK(cudaStreamSynchronize(c.s));
  if (loss_sum) *loss_sum = h;
  if (n_observed) *n_observed = hc;
  return NEF_OK;
}

int nef_loss(nef_plan_t plan, const float* Y, const uint8_t* mask, double alpha, double beta, float* const* factors,
             double* loss_sum, int64_t* n_observed, void* workspace, size_t ws_bytes, void* stream) {
  const nef_loss_spec ls = ab_spec(alpha, beta);
  return nef_loss_ex(plan, Y, mask, &ls, factors, loss_sum, n_observed, workspace, ws_bytes, stream);
}

size_t nef_host_scratch_bytes(nef_plan_t plan, int has_mask) {
  if (!plan) return 0;
  const nef::Plan& p = plan->p;
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  size_t b = al((size_t)p.n_local * 4);
  if (has_mask) b += al((size_t)p.n_local);
  for (auto& s : p.fshape) {
    size_t n = 1;
    for (auto d : s) n *= (size_t)d;
    b += al(n * 4);
  }
  return b + al(p.ws_bytes);
}

int nef_fit_host(nef_plan_t plan, const float* Y_host, const uint8_t* mask_host, double alpha, double beta, double eps,
                 float* const* factors_host, int iters, double* loss_trace, void* device_scratch, size_t scratch_bytes,
                 void* stream) {
  if (!plan || !Y_host || !factors_host || !device_scratch) return fail(NEF_E_ARG, "null argument");
  const nef::Plan& p = plan->p;
  if (scratch_bytes < nef_host_scratch_bytes(plan, mask_host != nullptr)) return fail(NEF_E_ARG, "device scratch too small");
  if (reinterpret_cast<uintptr_t>(device_scratch) & 255) return fail(NEF_E_ARG, "device scratch must be 256-byte aligned");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto al = [](size_t b) { return (b + 255) / 256 * 256; };
  char* d = static_cast<char*>(device_scratch);
  float* Yd = reinterpret_cast<float*>(d);
  d += al((size_t)p.n_local * 4);
  uint8_t* Md = nullptr;
  if (mask_host) { Md = reinterpret_cast<uint8_t*>(d); d += al((size_t)p.n_local); }
  std::vector<float*> Fd;
  std::vector<size_t> fn;
  for (auto& sh : p.fshape) {
    size_t n = 1;
    for (auto x : sh) n *= (size_t)x;
    Fd.push_back(reinterpret_cast<float*>(d));
    fn.push_back(n);
    d += al(n * 4);
  }
  CK(cudaMemcpyAsync(Yd, Y_host, (size_t)p.n_local * 4, cudaMemcpyHostToDevice, s));
  if (Md) CK(cudaMemcpyAsync(Md, mask_host, (size_t)p.n_local, cudaMemcpyHostToDevice, s));
  for (size_t l = 0; l < Fd.size(); ++l) CK(cudaMemcpyAsync(Fd[l], factors_host[l], fn[l] * 4, cudaMemcpyHostToDevice, s));
  int st = nef_fit(plan, Yd, Md, alpha, beta, eps, Fd.data(), iters, loss_trace, d, p.ws_bytes, stream);
  if (st) return st;
  for (size_t l = 0; l < Fd.size(); ++l) CK(cudaMemcpyAsync(factors_host[l], Fd[l], fn[l] * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return NEF_OK;
}

int nef_nccl_unique_id(void* out128) {
  if (!out128) return fail(NEF_E_ARG, "null out");
  std::string err;
  if (!load_nccl(err)) return fail(NEF_E_NCCL, err);
  int r = g_nccl.GetUniqueId(out128);
  if (r != 0) return fail(NEF_E_NCCL, "ncclGetUniqueId failed");
  return NEF_OK;
}

static int shard_impl(nef_plan_t plan, int rank, int world, const void* uid, bool host_only);

int nef_plan_shard(nef_plan_t plan, int rank, int world, const void* uid) {
  return shard_impl(plan, rank, world, uid, false);
}

int nef_plan_shard_host(nef_plan_t plan, int rank, int world) { return shard_impl(plan, rank, world, nullptr, true); }

static int shard_impl(nef_plan_t plan, int rank, int world, const void* uid, bool host_only) {
  if (!plan) return fail(NEF_E_ARG, "null plan");
  if (world < 1 || rank < 0 || rank >= world) return fail(NEF_E_ARG, "bad rank/world");
  nef::Plan& p = plan->p;
  if (p.shard_mode >= 0) return fail(NEF_E_ARG, "plan already sharded");
  // shard mode: largest (ties -> outermost)
  int sm = 0;
  for (int m = 1; m < (int)p.gshape.size(); ++m)
    if (p.gshape[m] > p.gshape[sm]) sm = m;
  int64_t n = p.gshape[sm];
  if (n < world) return fail(NEF_E_SHAPE, "largest mode smaller than world size");
  int64_t q = n / world, r = n % world;
  int64_t begin = rank * q + std::min<int64_t>(rank, r);
  int64_t len = q + (rank < r ? 1 : 0);
  const bool force = world == 1 && std::getenv("NEF_NCCL_FORCE") && std::getenv("NEF_NCCL_FORCE")[0] == '1';
  if ((world > 1 || force) && !host_only) {
    if (!uid) return fail(NEF_E_ARG, "null NCCL unique id");
    std::string err;
    if (!load_nccl(err)) return fail(NEF_E_NCCL, err);
    Uid u;
    std::memcpy(u.internal, uid, 128);
    void* comm = nullptr;
    int rr = g_nccl.CommInitRank(&comm, world, u, rank);
    if (rr != 0) return fail(NEF_E_NCCL, "ncclCommInitRank failed");
    p.nccl_comm = comm;
  }
  p.shard_mode = sm;
  p.rank = rank;
  p.world = world;
  p.local_begin = begin;
  p.local_len = len;
  p.shape = p.gshape;
  p.shape[sm] = len;
  char letter = p.out[sm];
  for (size_t l = 0; l < p.ops.size(); ++l) p.factor_has_shard[l] = p.ops[l].find(letter) != std::string::npos;
  std::string err;
  int st = nef::relower(p, err);
  if (st) return fail(st, err);
  return NEF_OK;
}

}  // extern "C"
