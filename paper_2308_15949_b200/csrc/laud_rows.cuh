// Row enumeration shared by the conv engines (tcgen05 bf16 and SIMT fp32):
// GEMM row m -> output pixel for dense grids, active-patch lists (m = p*S*S +
// local, reference.py:389-402 patch order) and pixel lists.
#pragma once
#include "laud_conv.cuh"

namespace laud {

struct RowPos {
  int n, y, x;
  int pix;  // linear output pixel (n*out_h + y)*out_w + x
};

// cell of patch-list position idx (list_expand: an entry covers list_expand cells)
__device__ __forceinline__ int list_cell(const ConvParams& p, int idx) {
  if (p.list_expand > 1) {
    const int e = idx / p.list_expand;
    return __ldg(p.list + e) * p.list_expand + (idx - e * p.list_expand);
  }
  return __ldg(p.list + idx);
}

__device__ __forceinline__ int rows_valid(const ConvParams& p) {
  if (p.row_mode == ROWS_DENSE || p.count == nullptr) return p.rows_max;
  int c = __ldg(p.count);
  if (p.list_expand > 1) c *= p.list_expand;
  long long r = (p.row_mode == ROWS_PATCH) ? (long long)c * p.patch_h * p.patch_w : (long long)c;
  return r < p.rows_max ? (int)r : p.rows_max;
}

// Output pixel of row m; false when the row is past the valid count.
__device__ __forceinline__ bool map_row(const ConvParams& p, int m, int nvalid, RowPos& o,
                                        bool& first_patch) {
  first_patch = false;
  if (m >= nvalid) return false;
  int hw = p.out_h * p.out_w;
  if (p.row_mode == ROWS_PATCH) {
    int s2 = p.patch_h * p.patch_w;
    int pi = m / s2;
    int l = m - pi * s2;
    int cell = list_cell(p, pi);
    int cpi = p.cells_h * p.cells_w;
    o.n = cell / cpi;
    int c = cell - o.n * cpi;
    int ci = c / p.cells_w;
    int cj = c - ci * p.cells_w;
    int ly = l / p.patch_w;
    o.y = ci * p.patch_h + ly;
    o.x = cj * p.patch_w + (l - ly * p.patch_w);
    o.pix = (o.n * p.out_h + o.y) * p.out_w + o.x;
    first_patch = (pi == 0);
    return true;
  }
  int pix;
  if (p.sample_rows > 0) {  // per-sample padded rows: one sample per M tile range
    const int smp = m / p.sample_rows;
    const int loc = m - smp * p.sample_rows;
    if (loc >= hw) return false;
    pix = smp * hw + loc;
  } else {
    pix = (p.row_mode == ROWS_PIXEL) ? __ldg(p.list + m) : m;
  }
  o.pix = pix;
  o.n = pix / hw;
  int r = pix - o.n * hw;
  o.y = r / p.out_w;
  o.x = r - o.y * p.out_w;
  return true;
}

}  // namespace laud
