// Host interface of the tcgen05 streaming kernel (kernels_tc.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"
#include "nef_internal.h"

namespace nef {
namespace tc {

struct TcArgs {
  int layout;                 // 0: rows innermost {R, CO}; 1: {CI, R}; 2: {CI, R, CO}
  int has_mask;
  int64_t R, CI, CO;          // merged extents (elements)
  int64_t tiles_inner;        // 64-wide tiles along CI (layouts 1, 2)
  int64_t tiles;              // total column tiles
  int64_t tiles_per_chunk;
  int K, KB;                  // bond and padded bond (32 | 64)
  int64_t n_rows;             // = R
  const float* U;             // [n_rows][K]
  int nc;                     // column modes (linear column index unravel)
  int64_t cdim[kMaxModes];
  int ntab;
  const float* tab[kMaxTabs];
  int64_t tcs[kMaxTabs][kMaxModes];
  int32_t boff[kMaxTabs][64];
  float* Qpart;               // [chunks][n_groups][2][n_rows][K]
  double* losspart;           // [row_blocks * chunks]
  long long* countpart;
  // batched restarts (N4): launch z index rs runs restart rs on the same Y tiles (its CTAs
  // stream the tiles the rs = 0 CTAs of the same (row block, chunk) fetch, from L2).  Index 0 is
  // the fields above; direct-V launches only.
  int nrs;
  const float* Ur[kMaxRestarts];
  const float* tabr[kMaxRestarts][kMaxTabs];
  float* Qpartr[kMaxRestarts];
  double* losspartr[kMaxRestarts];
  long long* countpartr[kMaxRestarts];
  const float* vdr[kMaxRestarts];   // direct-V table rows per restart (tensor map source)
  DivParams dv;
  int mode;                   // 0 update, 1 update + loss, 2 loss only
  float* debug;               // optional debug dump (first tile of CTA (0,0))
  long long* trace;           // optional pipeline timeline of CTA (0,0): [tile][16] clock64 stamps
  int vec4;                   // 1: every table has the bond contiguous (boff[k] = k), K % 4 == 0 and
                              //    16-byte aligned rows -> float4 V generation
  // direct V: the 64 columns of every tile are 64 consecutive rows of ONE
  // column table (the one holding the innermost column mode; every other table is constant
  // across a tile); those rows are TMA-loaded into the V stage and scaled in place.
  int vdirect;
  int var_tab;                // index of that table
  int64_t var_rows;           // its number of rows (row length = K)
  int64_t vd_E;               // run length: columns per run of consecutive table rows
  int64_t vd_tpr;             // tiles per run
  int64_t vd_pitch;           // row pitch (elements) of vd_rows_ptr (K rounded up to 4)
  const float* vd_rows_ptr;   // the table rows the TMA reads (the table, or its padded copy)
  int y3d;                    // layout 1 with CI % 32 == 0: Y tile = ONE 3-D TMA box {32, 2, 128}
                              //   over the view {32, CI/32, R} (both 128-byte halves of a row
                              //   requested back to back), smem [row][half][32] SW128
  int lconst;                 // loss passes accumulate only the factor-dependent part (R25):
                              //   LossOff<KIND>, the data-only sum comes from the sentinel pass
  int absy;                   // MM = 0 on raw unmasked Y: every entry observed, sign bits ignored
                              //   (an observed -0.0 is zero, not the sentinel's "missing")
  int split;                  // MM = 1 with labels 0..3 (R29): train = 1; loss partials per role [3][parts]
  int64_t n_groups;           // drain groups per chunk: Qpart is [chunks][n_groups][2][n_rows][K]

};

size_t smem_bytes(int mm, int kb);   // mm: 1 = uint8 mask stream, 2 = parameter stream, 0 = none; kb: 32 | 64
// aux: per-entry loss parameter (NB phi_i / binomial n_i), Y's layout, streamed as a second TMA
// ring (MM = 2; with the sentinel copy or unmasked Y only)
cudaError_t launch(const TcArgs& args, const float* Y, const uint8_t* M, int64_t row_blocks, int64_t chunks,
                   cudaStream_t s, const float* aux = nullptr);

}  // namespace tc
}  // namespace nef
