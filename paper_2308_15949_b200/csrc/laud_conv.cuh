// Parameter block of the implicit-GEMM convolution engine (conv_gemm.cu).
//
// One engine covers every convolution of the LAUDNet block path:
//   rows    m  = output pixels, enumerated densely, from a patch list
//               (m = p*S*S + local), or from a pixel list;
//   A[m, k] = act[input pixel of (row m, tap t)][channel c], k = t*Kpad + c,
//             gathered by cp.async with zero fill outside the image;
//   B[n, k] = packed weights [Cout][taps][Kpad] (TMA, 128B swizzle);
//   D       = tcgen05 fp32 accumulator in TMEM, epilogue: scale/bias/ReLU,
//             optional residual add, bf16 (or fp32) store to the row's
//             destination (scattered pixel or compact row).
#pragma once
#include <cstdint>

namespace laud {

enum RowMode : int { ROWS_DENSE = 0, ROWS_PATCH = 1, ROWS_PIXEL = 2 };
enum OutMode : int { OUT_PIXEL = 0, OUT_ROW = 1 };
enum BGather : int { B_BOX = 0, B_GATHER_N = 1, B_GATHER_K = 2 };

struct ConvParams {
  // ---- rows (output pixels)
  int row_mode;          // RowMode
  const int* list;       // patch list (cell index) or pixel list (pixel index)
  int list_expand;       // > 1: each list entry e stands for cells e*k .. e*k+k-1 (k = list_expand;
                         // layer blocks: a sample list read as its S x S cells), count scales by k
  const int* count;      // device count of list entries; nullptr -> use rows_max
  int rows_max;          // upper bound on rows (grid sizing)
  int batch;             // N
  int out_h, out_w;      // output grid
  int patch_h, patch_w;  // S x S patch (ROWS_PATCH); H x W of the image in layer mode
  int cells_h, cells_w;  // out_h/patch_h, out_w/patch_w
  // ---- A operand
  const void* act;       // bf16 NHWC input
  int in_h, in_w;        // input grid
  int in_c;              // valid channels (multiple of 8)
  int in_ld;             // elements per pixel row (>= in_c, multiple of 8)
  int a_compact;         // 1: A row = m directly (1x1, taps must be 1)
  int a_tma;             // 1: A rows gathered with TMA tile::gather4 (else cp.async)
  int a_tile;            // 1: the 128 A rows of a tile are contiguous: one 2D TMA box
  int a_box;             // 1: S x S patch rows loaded as one 4D TMA box per patch and tap
  // fused masker (dense 1x1 conv1 with contiguous A rows, a_tile): idle producer
  // warps read each A stage from smem and store dot(x_row, adot_w) per row
  // (= per dense input pixel) into adot_out[row]; the decision pass sums the
  // cell windows in a fixed order
  const float* adot_w;
  int tma_out;  // kPlain epilogues: 1 = dense rows stored as 32-row TMA boxes, 2 = S x S patch boxes (4D)
  float* adot_out;
  int a_rows;            // rows of the A tensor map (also the out-of-bounds marker)
  int ksize, stride, pad;
  int kpad;              // in_c rounded up to 64 (+64 for grouped convs)
  int groups;            // > 1: block-diagonal weights; per N tile a K window of its groups
  int gw_in, gw_out;     // channels per group (input, output)
  int num_kb;            // ksize*ksize*kpad/64
  // ---- output
  int n_out;             // output channels (multiple of 8)
  const float* scale;    // per-channel, nullable
  const float* bias;     // per-channel, nullable
  int relu;              // ReLU after scale/bias (and after residual add if resid)
  int out_mode;          // OutMode
  void* out;             // bf16 (or fp32 when out_f32) destination
  int out_ld;            // elements per destination row
  int out_f32;           // store fp32 instead of bf16
  const void* resid;     // bf16 residual (read at the destination pixel), nullable
  int resid_ld;
  // ---- ReLU only where the destination pixel's cell is inactive (skip path of
  //      a downsample block under a spatial mask): coarse[cell] == 0 -> ReLU.
  const unsigned char* relu_inactive_coarse;
  // ---- dense-masked (training-style) semantics, `reference.py:313-353`:
  //      y *= coarse[cell of the destination pixel]   (spatial / layer), and
  //      y *= chmask[n][channel]                      (channel, per sample).
  const unsigned char* ymask_coarse;
  const unsigned char* ymask_channel;
  // ---- per-sample dynamic width (channel skipping, `reference.py:404-423`)
  int sample_rows;         // >0: rows padded per sample (multiple of 128), one sample per tile
  const int* chan_count;   // [N] kept channels k_n
  int n_dyn;               // output columns >= k_n are skipped (N ragged)
  int k_dyn;               // K per tap = roundup(k_n, 64) (K ragged)
  int b_batched;           // B is [N][n_out][K] (3D tensor map, sample coordinate)
  const int* col_index;    // [N][col_index_ld]: scale/bias index of output column c
  int col_index_ld;
  // ---- weights gathered in-kernel per sample (channel skipping at large batch):
  //      B_GATHER_N: B rows = weight rows b_index[sample][n0 + j] (cp.async,
  //                  K-major [rows][taps * kpad]; j >= k_n -> zero rows);
  //      B_GATHER_K: B = weightT rows b_index[sample][k] for the tile's 64 K
  //                  (MN-major [K rows][n_out], 1x1 only; k >= k_n -> zero).
  int b_gather;
  const int* b_index;
  int b_index_ld;
  int b_rows;              // rows of the gathered weight tensor
  const void* weight_g;    // gathered weights (bf16) and their row stride in elements
  int b_ld;
  // ---- split-K over a thread-block cluster (halo patch conv, small grids):
  //      ksplit CTAs of a cluster take disjoint channel-block ranges of one
  //      tile; fp32 partials are reduced through distributed shared memory
  int ksplit;
  int tail_split;          // halo conv, large grids: the last partial wave's tiles split over 2-CTA clusters
  // ---- masker-conv3 fusion: mdot_out[cell(row)] += dot(bf16 output row, mdot_w)
  const float* mdot_w;
  float* mdot_out;
  // ---- fault hook (tests only): shift the first patch's destination one cell
  int misplace_first;
  // ---- debug timeline (laud_debug_set_trace): CTA 0 records %globaltimer at
  //      pipeline events; nullptr (always, outside tools/) = off
  unsigned long long* trace;
  const void* weight_f32;  // fp32 mode: packed fp32 weights (conv_f32.cu)
  int dbg;  // debug ablations (LAUD_DBG, tools only): 1 no math, 2 no stores, 4 no TMEM loads,
           // 8 no A loads, 16 no B loads
};

// trace slots (CTA 0): MMA full-wait done per k-block, B-producer empty-wait
// done per k-block, A-producer (warp 0) empty-wait done per k-block, epilogue
// warp 4 per tile: acc_full done / stores done.
constexpr int TRACE_MMA = 0, TRACE_B = 4096, TRACE_A = 8192, TRACE_EPI = 12288, TRACE_SLOTS = 16384;

}  // namespace laud
