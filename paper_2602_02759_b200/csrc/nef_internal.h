// Internal structures shared by the planner (host C++) and the kernels (CUDA).
// See DESIGN.md §Planner for the lowering these describe.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

namespace nef {

constexpr int kMaxDims = 8;      // max indices per operand / per einsum step side
constexpr int kMaxTabs = 4;      // max KR tables on the column side of a lowering
constexpr int kMaxModes = 8;     // max observed modes
constexpr int kMaxRestarts = 4;  // restarts sharing one streamed pass (N4)
constexpr int kSentParts = 148 * 16 + 1;   // sentinel pass block partials (kernels.h kSentBlocks + 1)
// tcgen05 path: the tensor core's fp32 accumulation truncates, so the numerator / denominator
// accumulators are drained to separate split partials every kDrainTiles tiles (<= 2048
// truncating accumulation steps per partial; summed in fp64 by reduce_q)
constexpr int kDrainTiles = 256;
// tcgen05 path only for factors whose entries each sum at least this many Y entries (R26)
constexpr int64_t kTcMinSlab = 2048;

// ---------------------------------------------------------------------------------
// Small einsum engine: C[out] = sum_{sum} A[...] * B[...]   (B optional)
// Buffers are referred to by id; ids < 0x100 are factors, others workspace regions.
// ---------------------------------------------------------------------------------
enum BufKind : int { BUF_FACTOR = 0, BUF_WS = 1, BUF_NONE = 2 };

struct BufRef {
  int kind = BUF_NONE;   // BufKind
  int64_t id = -1;       // factor index, or byte offset in the workspace
  int64_t elems = 0;
};

struct EinStep {
  BufRef a, b, c;                    // b.kind == BUF_NONE -> unary
  std::string a_idx, b_idx, c_idx;   // index strings (for description / debug executor)
  int nout = 0;
  int64_t odim[kMaxDims] = {};
  int64_t as_o[kMaxDims] = {}, bs_o[kMaxDims] = {};
  int nsum = 0;
  int64_t sdim[kMaxDims] = {};
  int64_t as_s[kMaxDims] = {}, bs_s[kMaxDims] = {};
  int64_t out_size = 1, sum_size = 1;
};

// fp32 scratch floats a GEMM-shaped step needs for its split partials (0: none; kernels_ffma.cu)
int64_t einstep_scratch_floats(const EinStep& st);

struct EinProgram {
  std::vector<EinStep> steps;     // executed in order; last step writes the result
  BufRef result;                  // where the result lives (may alias an input when steps empty)
  std::string result_idx;
  double macs = 0;                // cost estimate
};

// ---------------------------------------------------------------------------------
// Lowering of one factor update
//   Yhat[row, col] = sum_b U[row, b] * V[col, b],  V[col, b] = prod_t T_t[col_t, b_t]
//   Q_a[row, b] = sum_col a(Y, Yhat)[row, col] V[col, b]   (and Q_b with b(Y, Yhat))
//   Num_ell = epilogue(Q_a, row-side factors except ell)    (= einsum(swap(rowmodel, ell)))
// ---------------------------------------------------------------------------------
struct ColTable {
  EinProgram prog;          // computes the table; result index order = (its col modes, its bond idx)
  std::string idx;          // table index string
  int64_t cstride[kMaxModes] = {};   // stride per column mode (0 if the table lacks it)
  std::vector<int32_t> boff;         // offset per linear bond index b in [0, K)
};

struct Lowering {
  int ell = -1;
  std::vector<int> row_modes, col_modes;   // Y modes (positions in the output string), Y order
  std::string row_idx, col_idx;            // letters of those modes
  std::string bond;                        // bond index letters (order = linear bond index, last fastest)
  int64_t K = 1;                           // bond size
  int64_t n_rows = 1, n_cols = 1;
  int64_t rdim[kMaxModes] = {}, rystride[kMaxModes] = {};   // row unravel dims / Y strides
  int64_t cdim[kMaxModes] = {}, cystride[kMaxModes] = {};   // col unravel dims / Y strides
  bool row_fast = false;                   // innermost Y mode lies on the row side
  EinProgram uprog;                        // U[row, bond] (result idx = row_idx + bond)
  std::vector<ColTable> tabs;              // column tables
  EinProgram epi;                          // Num (factor ell's layout) from Q (+ row factors)
  bool epi_identity = false;
  std::vector<int> row_factors, col_factors;
  // workspace layout (byte offsets)
  int64_t ws_U = 0, ws_boff = 0, ws_Qpart = 0, ws_Q = 0, ws_num = 0, ws_den = 0, ws_tmp = 0;
  int64_t ws_losspart = 0;
  int64_t n_chunks = 1;                    // split of the column range (deterministic partials)
  int64_t ws_end = 0;
  double cost = 0;
  // tcgen05 path geometry (filled by the planner)
  bool tc_ok = false;
  bool tc_mask_ok = false;      // uint8 mask strides are TMA-legal too
  int tc_layout = 0;           // 0: rows innermost (2-D {R, CO}); 1: cols inner 2-D {CI, R}; 2: 3-D {CI, R, CO}
  int64_t tc_R = 0;             // merged row extent
  int64_t tc_CI = 1, tc_CO = 1; // merged inner / outer column extents
  int64_t tc_rstride = 0;       // Y element stride of the merged row dim
  int64_t tc_costride = 0;      // Y element stride of the merged outer column dim
  int tc_KB = 32;               // padded bond (32 or 64)
  int64_t tc_tiles = 0;         // column tiles (64 wide)
  int64_t tc_chunks = 1;        // split of the tile range per row block
  int64_t tc_row_blocks = 0;    // 128-row blocks
  int64_t tc_groups = 1;        // drain groups per chunk (kDrainTiles tiles each)
  int64_t ws_tc_Qpart = 0;      // partial buffer for the tcgen05 path
  int64_t ws_tc_losspart = 0;   // per-CTA loss / count partials of the tcgen05 path
  // direct V: one table vd_tab holds the trailing column modes as consecutive
  // rows (row pitch K), every other table is constant over them; runs of vd_E columns map to
  // consecutive table rows, and no 64-column tile straddles two runs
  int vd_tab = -1;
  int64_t vd_E = 0;
  int64_t vd_rows = 0;          // rows of that table
  int64_t vd_Kp = 0;            // TMA row pitch (elements): K rounded up to 4
  int64_t ws_vpad = -1;         // padded copy of the table when K % 4 != 0 (else -1)
  bool tabs_merged = false;     // all column factors merged into one table (small column space)
  std::vector<std::pair<int64_t, int64_t>> ws_allocs;   // every workspace region [offset, end) it uses
  // inside a sweep (updates in order 0, 1, ...): U / table q are the result an earlier update
  // of the same sweep left in the workspace (planner: sweep_reuse)
  bool reuse_u = false;
  std::vector<char> reuse_tab;
  BufRef alias_u;                  // where the reused result lives
  std::vector<BufRef> alias_tab;
};

struct Plan {
  std::string model;                 // normalized string
  std::vector<std::string> ops;      // operand subscripts
  std::string out;                   // output subscripts
  std::vector<int64_t> gshape;       // global Y shape
  std::vector<int64_t> shape;        // local Y shape
  int64_t dims[128] = {};            // size per ASCII letter
  std::vector<std::vector<int64_t>> fshape;   // local factor shapes
  std::vector<std::string> einstr;   // swap(model, ell)
  std::vector<Lowering> low;         // per factor
  int64_t n_local = 0;               // local entries
  size_t ws_bytes = 0;
  int64_t ws_trace = 0;              // fp64 trace accumulators
  int64_t ws_dterm = 0;              // [double][long long]: data-only loss sum, observed count (R25)
  int64_t ws_dpart = 0;              // their kSentParts block partials (doubles, then counts)
  int64_t ws_fsave = 0;              // factor copies of nef_fit_split (iterate entering a sweep)
  int64_t ws_sent = 0;               // NaN-sentinel copy of Y (nef_fit with a mask)
  int64_t ws_escr = 0;               // split partials of GEMM-shaped einsum steps (launch_einstep)
  // sharding
  int shard_mode = -1, rank = 0, world = 1;
  int64_t local_begin = 0, local_len = 0;
  void* nccl_comm = nullptr;
  std::vector<bool> factor_has_shard;
  int num_sms = 148;
};

// planner entry points (plan.cpp)
int build_plan(const char* einsum, int n_modes, const int64_t* shape, int n_ranks, const int64_t* ranks,
               Plan& p, std::string& err);
int relower(Plan& p, std::string& err);           // recompute lowerings after sharding
std::string describe_plan(const Plan& p);

}  // namespace nef
