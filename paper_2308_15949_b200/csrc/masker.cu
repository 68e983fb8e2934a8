// Spatial / layer masker and stable stream compaction (sm_100a).
//
// K1a cell_dot_kernel   d[cell] partials = sum over the cell's (stride*S)^2 input
//                       pixels of x . (W0 - W1)  — the fused-masker identity of
//                       `reference.py:244-253` applied to the pooled 1x1 conv of
//                       `reference.py:173-174`.  128-bit NHWC loads, one warp per
//                       (cell, split) work item, deterministic split partials.
// K1b compact_kernel    decision = mean(d) + bias >= 0 (compute wins ties,
//                       `reference.py:183`), then a warp-ballot/shuffle block scan
//                       and decoupled look-back across CTAs to emit the active
//                       cell indices in row-major order — identical to
//                       `np.argwhere` in `build_gather_plan` (`reference.py:133-135`)
//                       — plus the device-side count (no host sync).
// The same compaction core emits the conv1 pixel set (union of the active
// patches' 3x3 halo windows on the input grid) and lists from given masks.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>

#include "laud_launch.cuh"
#include "laud_ptx.cuh"

namespace laud {

constexpr int CT_THREADS = 256;
constexpr int CT_ITEMS = 1;
constexpr int CT_TILE = CT_THREADS * CT_ITEMS;  // 256 items per CTA: wide grids beat short look-back chains (measured)

// Look-back scratch; zero at allocation, restored to zero by the last CTA.
struct ScanState {
  unsigned int tile_ctr;
  unsigned int done_ctr;
  unsigned int pad[2];
  unsigned long long tiles[1];  // [num_tiles]
};

constexpr unsigned long long FLAG_AGG = 1ull << 32;
constexpr unsigned long long FLAG_INC = 2ull << 32;

// ---------------------------------------------------------------------------
// K1a: per (cell, split) partial dot products
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ float dot8(const T* p, const float* w);
template <>
__device__ __forceinline__ float dot8<__nv_bfloat16>(const __nv_bfloat16* p, const float* w) {
  const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
  float a = 0.f;
  float2 f;
  f = unpack_bf16x2(v.x); a = fmaf(f.x, w[0], a); a = fmaf(f.y, w[1], a);
  f = unpack_bf16x2(v.y); a = fmaf(f.x, w[2], a); a = fmaf(f.y, w[3], a);
  f = unpack_bf16x2(v.z); a = fmaf(f.x, w[4], a); a = fmaf(f.y, w[5], a);
  f = unpack_bf16x2(v.w); a = fmaf(f.x, w[6], a); a = fmaf(f.y, w[7], a);
  return a;
}
template <>
__device__ __forceinline__ float dot8<float>(const float* p, const float* w) {
  const float4 u = __ldg(reinterpret_cast<const float4*>(p));
  const float4 v = __ldg(reinterpret_cast<const float4*>(p) + 1);
  float a = 0.f;
  a = fmaf(u.x, w[0], a); a = fmaf(u.y, w[1], a); a = fmaf(u.z, w[2], a); a = fmaf(u.w, w[3], a);
  a = fmaf(v.x, w[4], a); a = fmaf(v.y, w[5], a); a = fmaf(v.z, w[6], a); a = fmaf(v.w, w[7], a);
  return a;
}

template <typename T>
__global__ void __launch_bounds__(256) cell_dot_kernel(
    const T* __restrict__ x, int ld, int n, int h, int w, int c, int win, int cells_h,
    int cells_w, const float* __restrict__ wdiff, int splits, int chunks_per_split,
    float* __restrict__ partial, const uint8_t* __restrict__ prev_coarse, float* __restrict__ dn) {
  pdl_wait();  // PDL: predecessors' outputs visible from here
  pdl_trigger();
  extern __shared__ float s_w[];
  for (int i = threadIdx.x; i < c; i += blockDim.x) s_w[i] = wdiff[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cpp = c >> 3;  // 8-channel chunks per pixel
  const int cell_chunks = win * win * cpp;
  const long long items = (long long)n * cells_h * cells_w * splits;
  const long long item = (long long)blockIdx.x * (blockDim.x >> 5) + warp;
  if (item >= items) return;
  const int cell = (int)(item / splits);
  const int split = (int)(item - (long long)cell * splits);
  const int cpi = cells_h * cells_w;
  const int ni = cell / cpi;
  const int cr = cell - ni * cpi;
  const int ci = cr / cells_w, cj = cr - (cr / cells_w) * cells_w;
  const int q0 = split * chunks_per_split;
  int q1 = min(q0 + chunks_per_split, cell_chunks);
  float acc = 0.f;
  // masker-conv3 fusion: cells the previous block computed already carry their
  // dot product (accumulated by that block's conv3 epilogue) in dn; only cells
  // it skipped are read from x.  dn is consumed (zeroed) for the next block.
  if (dn) {
    const bool prev_active = prev_coarse && prev_coarse[cell];
    if (prev_active) q1 = q0;  // skip the loads
    if (split == 0 && lane == 0) {
      if (prev_active) acc = dn[cell];
      dn[cell] = 0.f;
    }
  }
#pragma unroll 4
  for (int q = q0 + lane; q < q1; q += 32) {
    const int px = q / cpp;
    const int ch = (q - px * cpp) << 3;
    const int py = px / win;
    const int pxx = px - py * win;
    const int yy = ci * win + py, xx = cj * win + pxx;
    acc += dot8<T>(x + ((size_t)(ni * h + yy) * w + xx) * ld + ch, s_w + ch);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) partial[item] = acc;
}

// Layer masker (one cell = the whole image; contiguous NHWC rows, C = 256 P):
// a split is 1024 consecutive 16-byte chunks of the image, so lane l always
// meets channel chunk l + 32 j at step j mod P — the weights stay in
// registers, no index arithmetic per load, P independent accumulators added
// in j order at the end (deterministic).
template <int P>
__global__ void __launch_bounds__(256) cell_dot_contig_kernel(const __nv_bfloat16* __restrict__ x, int cell_chunks,
                                                              const float* __restrict__ wdiff, int splits,
                                                              float* __restrict__ partial, long long items) {
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long item = (long long)blockIdx.x * 8 + warp;
  if (item >= items) return;
  const long long cell = item / splits;
  const int split = (int)(item - cell * splits);
  float wv[P][8];
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(wdiff + (lane + 32 * j) * 8));
    const float4 b = __ldg(reinterpret_cast<const float4*>(wdiff + (lane + 32 * j) * 8 + 4));
    wv[j][0] = a.x; wv[j][1] = a.y; wv[j][2] = a.z; wv[j][3] = a.w;
    wv[j][4] = b.x; wv[j][5] = b.y; wv[j][6] = b.z; wv[j][7] = b.w;
  }
  const uint4* src = reinterpret_cast<const uint4*>(x) + cell * cell_chunks + (long long)split * 1024;
  const int nq = min(1024, cell_chunks - split * 1024);
  float acc[P];
#pragma unroll
  for (int j = 0; j < P; ++j) acc[j] = 0.f;
#pragma unroll 2
  for (int q0 = lane; q0 < nq; q0 += 32 * P) {
    uint4 v[P];
#pragma unroll
    for (int j = 0; j < P; ++j) v[j] = q0 + 32 * j < nq ? __ldg(src + q0 + 32 * j) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
    for (int j = 0; j < P; ++j) {
      float2 f;
      f = unpack_bf16x2(v[j].x); acc[j] = fmaf(f.x, wv[j][0], acc[j]); acc[j] = fmaf(f.y, wv[j][1], acc[j]);
      f = unpack_bf16x2(v[j].y); acc[j] = fmaf(f.x, wv[j][2], acc[j]); acc[j] = fmaf(f.y, wv[j][3], acc[j]);
      f = unpack_bf16x2(v[j].z); acc[j] = fmaf(f.x, wv[j][4], acc[j]); acc[j] = fmaf(f.y, wv[j][5], acc[j]);
      f = unpack_bf16x2(v[j].w); acc[j] = fmaf(f.x, wv[j][6], acc[j]); acc[j] = fmaf(f.y, wv[j][7], acc[j]);
    }
  }
  float a = 0.f;
#pragma unroll
  for (int j = 0; j < P; ++j) a += acc[j];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if (lane == 0) partial[item] = a;
}

// Same as cell_dot_kernel for cells of <= 32*NPL chunks (one split): every
// lane issues all of its NPL 16-byte loads before the first FMA, so a warp
// keeps a whole cell (up to 8 KiB) in flight.
template <int NPL>
__global__ void __launch_bounds__(256) cell_dot_unrolled_kernel(
    const __nv_bfloat16* __restrict__ x, int ld, int n, int h, int w, int c, int win, int cells_h,
    int cells_w, const float* __restrict__ wdiff, float* __restrict__ partial) {
  extern __shared__ float s_w[];
  for (int i = threadIdx.x; i < c; i += blockDim.x) s_w[i] = wdiff[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cpp = c >> 3;
  const int cell_chunks = win * win * cpp;
  const int total = n * cells_h * cells_w;
  const int cell = blockIdx.x * (blockDim.x >> 5) + warp;
  if (cell >= total) return;
  const int cpi = cells_h * cells_w;
  const int ni = cell / cpi;
  const int cr = cell - ni * cpi;
  const int ci = cr / cells_w, cj = cr - (cr / cells_w) * cells_w;
  uint4 v[NPL];
  int chv[NPL];
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int q = lane + 32 * i;
    chv[i] = -1;
    v[i] = make_uint4(0, 0, 0, 0);
    if (q < cell_chunks) {
      const int px = q / cpp;
      const int ch = (q - px * cpp) << 3;
      const int py = px / win;
      v[i] = __ldg(reinterpret_cast<const uint4*>(
          x + ((size_t)(ni * h + ci * win + py) * w + cj * win + (px - py * win)) * ld + ch));
      chv[i] = ch;
    }
  }
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    if (chv[i] < 0) continue;
    const float* ww = s_w + chv[i];
    float2 f;
    f = unpack_bf16x2(v[i].x); acc = fmaf(f.x, ww[0], acc); acc = fmaf(f.y, ww[1], acc);
    f = unpack_bf16x2(v[i].y); acc = fmaf(f.x, ww[2], acc); acc = fmaf(f.y, ww[3], acc);
    f = unpack_bf16x2(v[i].z); acc = fmaf(f.x, ww[4], acc); acc = fmaf(f.y, ww[5], acc);
    f = unpack_bf16x2(v[i].w); acc = fmaf(f.x, ww[6], acc); acc = fmaf(f.y, ww[7], acc);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) partial[cell] = acc;
}

// ---------------------------------------------------------------------------
// flag sources for the compaction core
// ---------------------------------------------------------------------------
struct MaskerFlag {  // decision from split partials; also materialises coarse
  const float* partial;
  int splits;
  float inv_area, bias;
  uint8_t* coarse;
  __device__ bool operator()(int i) const {
    float s = 0.f;
    for (int k = 0; k < splits; ++k) {
      s += partial[(size_t)i * splits + k];
    }
    const bool f = s * inv_area + bias >= 0.f;
    if (coarse) coarse[i] = f ? 1 : 0;
    return f;
  }
};

// Conv1-fused masker: per-pixel dots (one per dense conv1 row) summed over
// each cell's win x win input window in fixed row-major order (deterministic),
// then d = sum / win^2 + bias >= 0 (`reference.py:173-183`).
struct PixelWindowFlag {
  const float* dots;
  int h, w, win, cells_h, cells_w;
  float inv_area, bias;
  uint8_t* coarse;
  __device__ bool operator()(int i) const {
    const int cpi = cells_h * cells_w;
    const int ni = i / cpi;
    const int cr = i - ni * cpi;
    const int ci = cr / cells_w, cj = cr - (cr / cells_w) * cells_w;
    const float* base = dots + ((size_t)ni * h + ci * win) * w + cj * win;
    float s = 0.f;
    for (int py = 0; py < win; ++py)
      for (int px = 0; px < win; ++px) s += base[(size_t)py * w + px];
    const bool f = s * inv_area + bias >= 0.f;
    if (coarse) coarse[i] = f ? 1 : 0;
    return f;
  }
};

struct GivenFlag {  // list from a caller-supplied coarse mask
  const uint8_t* coarse;
  __device__ bool operator()(int i) const { return coarse[i] != 0; }
};

// conv1 work set: input pixel needed iff an active cell's conv2 input window
// [ci*S*st - 1, ci*S*st + (S-1)*st + 1] (rows and cols) covers it.
struct DilateFlag {
  const uint8_t* coarse;
  int h, w, s, st, cells_h, cells_w, radius;
  __device__ bool operator()(int i) const {
    const int hw = h * w;
    const int ni = i / hw;
    const int r = i - ni * hw;
    const int y = r / w, xx = r - (r / w) * w;
    const int ss = s * st;
    const int span = (s - 1) * st + radius;  // window: [ci*ss - radius, ci*ss + span]
    int ci0 = y - span;
    ci0 = ci0 <= 0 ? 0 : (ci0 + ss - 1) / ss;
    int ci1 = min((y + radius) / ss, cells_h - 1);
    int cj0 = xx - span;
    cj0 = cj0 <= 0 ? 0 : (cj0 + ss - 1) / ss;
    int cj1 = min((xx + radius) / ss, cells_w - 1);
    const uint8_t* cm = coarse + (size_t)ni * cells_h * cells_w;
    for (int ci = ci0; ci <= ci1; ++ci)
      for (int cj = cj0; cj <= cj1; ++cj)
        if (cm[ci * cells_w + cj]) return true;
    return false;
  }
};

// ---------------------------------------------------------------------------
// K1b: stable compaction with decoupled look-back
// ---------------------------------------------------------------------------
// Decoupled look-back, one warp: publish this tile's aggregate, then scan the
// predecessors 32 at a time (one lane each) until the nearest inclusive
// prefix; returns the exclusive prefix (same value in every lane).
__device__ __forceinline__ int warp_lookback(ScanState* st, int tile, int agg, int lane) {
  if (lane == 0)
    atomicExch(&st->tiles[tile], (tile == 0 ? FLAG_INC : FLAG_AGG) | (unsigned)agg);
  int excl = 0;
  if (tile > 0) {
    volatile unsigned long long* tiles = st->tiles;
    for (int j = tile - 1;; j -= 32) {
      const int idx = j - lane;  // lane 0 = nearest predecessor
      unsigned long long sw = FLAG_INC;
      if (idx >= 0) {
        do {
          sw = tiles[idx];
        } while ((sw >> 32) == 0);
      }
      const unsigned inc = __ballot_sync(0xffffffffu, (sw >> 32) == 2);
      const int stop = inc ? __ffs(inc) - 1 : 31;
      int v = (lane <= stop && idx >= 0) ? (int)(sw & 0xffffffffu) : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      excl += v;
      if (inc) break;
    }
    if (lane == 0) atomicExch(&st->tiles[tile], FLAG_INC | (unsigned)(excl + agg));
  }
  return excl;
}

// The last CTA to finish restores the look-back scratch for the next launch.
__device__ __forceinline__ void scan_state_release(ScanState* st, int num_tiles, int* s_flag) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned done = atomicAdd(&st->done_ctr, 1u);
    *s_flag = (done == (unsigned)num_tiles - 1) ? 1 : 0;
  }
  __syncthreads();
  if (*s_flag) {
    for (int i = threadIdx.x; i < num_tiles; i += blockDim.x) st->tiles[i] = 0ull;
    if (threadIdx.x == 0) {
      st->tile_ctr = 0;
      st->done_ctr = 0;
    }
    __threadfence();
  }
}

template <class Flag>
__global__ void __launch_bounds__(CT_THREADS) compact_kernel(Flag flag, int total,
                                                             int* __restrict__ list,
                                                             int* __restrict__ count,
                                                             ScanState* st, int num_tiles) {
  pdl_wait();  // PDL: predecessors' outputs visible from here
  pdl_trigger();
  __shared__ int s_tile;
  __shared__ int s_warp[CT_THREADS / 32];
  __shared__ int s_excl;
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(&st->tile_ctr, 1u);
  __syncthreads();
  const int tile = s_tile;
  const int base = tile * CT_TILE + threadIdx.x * CT_ITEMS;
  bool f[CT_ITEMS];
  int cnt = 0;
#pragma unroll
  for (int j = 0; j < CT_ITEMS; ++j) {
    f[j] = (base + j < total) ? flag(base + j) : false;
    cnt += f[j];
  }
  // block-wide exclusive scan of per-thread counts
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int v = lane < CT_THREADS / 32 ? s_warp[lane] : 0;
    int wi = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += u;
    }
    if (lane < CT_THREADS / 32) s_warp[lane] = wi - v;  // exclusive warp offsets
    const int agg = __shfl_sync(0xffffffffu, wi, CT_THREADS / 32 - 1);
    const int excl = warp_lookback(st, tile, agg, lane);
    if (lane == 0) {
      s_excl = excl;
      if (tile == num_tiles - 1) *count = excl + agg;
    }
  }
  __syncthreads();
  int pos = s_excl + s_warp[warp] + incl - cnt;
#pragma unroll
  for (int j = 0; j < CT_ITEMS; ++j)
    if (f[j]) list[pos++] = base + j;
  scan_state_release(st, num_tiles, &s_tile);
}

// ---------------------------------------------------------------------------
// K1 fused: masker dot products + decision + compaction in one pass over x
// (cells that fit one warp work item).  TC cells per CTA, one warp per cell.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256) masker_fused_kernel(
    const T* __restrict__ x, int ld, int n, int h, int w, int c, int win, int cells_h, int cells_w,
    const float* __restrict__ wdiff, float bias, float inv_area, int tc, uint8_t* __restrict__ coarse,
    float* __restrict__ dots, int* __restrict__ list, int* __restrict__ count, ScanState* st,
    int num_tiles) {
  pdl_wait();  // PDL: predecessors' outputs visible from here
  pdl_trigger();
  extern __shared__ float s_w[];           // c floats
  __shared__ unsigned char s_flag[256];
  __shared__ int s_tile, s_excl, s_rel;
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(&st->tile_ctr, 1u);
  for (int i = threadIdx.x; i < c; i += blockDim.x) s_w[i] = wdiff[i];
  __syncthreads();
  const int tile = s_tile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int total = n * cells_h * cells_w;
  const int cell0 = tile * tc;
  const int cpp = c >> 3;
  const int cell_chunks = win * win * cpp;
  const int cpi = cells_h * cells_w;
  // wpc warps per cell (8 / tc): each takes every wpc-th 64-chunk step of the
  // cell; the warps' sums are added in warp order (deterministic)
  const int wpc = 8 / tc, sub = warp % wpc;
  __shared__ float s_part[8];
  for (int lc = warp / wpc; lc < tc; lc += 8 / wpc) {
    const int cell = cell0 + lc;
    if (cell < total) {
      const int ni = cell / cpi;
      const int cr = cell - ni * cpi;
      const int ci = cr / cells_w, cj = cr - (cr / cells_w) * cells_w;
      float a0 = 0.f, a1 = 0.f;
#pragma unroll 4
      for (int q = lane + 64 * sub; q < cell_chunks; q += 64 * wpc) {
        const int px = q / cpp;
        const int ch = (q - px * cpp) << 3;
        const int py = px / win;
        a0 += dot8<T>(x + ((size_t)(ni * h + ci * win + py) * w + cj * win + (px - py * win)) * ld + ch,
                      s_w + ch);
        const int q2 = q + 32;
        if (q2 < cell_chunks) {
          const int px2 = q2 / cpp;
          const int ch2 = (q2 - px2 * cpp) << 3;
          const int py2 = px2 / win;
          a1 += dot8<T>(x + ((size_t)(ni * h + ci * win + py2) * w + cj * win + (px2 - py2 * win)) * ld + ch2,
                        s_w + ch2);
        }
      }
      float acc = a0 + a1;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) s_part[warp] = acc;
    }
  }
  __syncthreads();
  if (threadIdx.x < tc) {  // thread lc decides cell lc
    const int lc = threadIdx.x, cell = cell0 + lc;
    bool f = false;
    if (cell < total) {
      float acc = 0.f;
      for (int k = 0; k < wpc; ++k) acc += s_part[lc * wpc + k];
      f = acc * inv_area + bias >= 0.f;
      coarse[cell] = f ? 1 : 0;
      if (dots) dots[cell] = acc;
    }
    s_flag[lc] = f ? 1 : 0;
  }
  __syncthreads();
  // tile-local exclusive scan of tc (<= 256) flags: thread t owns flag t
  const bool mine = threadIdx.x < tc && s_flag[threadIdx.x];
  const unsigned bal = __ballot_sync(0xffffffffu, mine);
  __shared__ int s_wc[8];
  if (lane == 0) s_wc[warp] = __popc(bal);
  __syncthreads();
  if (warp == 0) {
    const int v = lane < 8 ? s_wc[lane] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane < 8) s_wc[lane] = incl - v;
    const int agg = __shfl_sync(0xffffffffu, incl, 7);
    const int excl = warp_lookback(st, tile, agg, lane);
    if (lane == 0) {
      s_excl = excl;
      if (tile == num_tiles - 1) *count = excl + agg;
    }
  }
  __syncthreads();
  if (mine) list[s_excl + s_wc[warp] + __popc(bal & ((1u << lane) - 1u))] = cell0 + threadIdx.x;
  scan_state_release(st, num_tiles, &s_rel);
}

// ---------------------------------------------------------------------------
// K1 strip masker: one CTA streams one row of cells (win image rows x W x C,
// contiguous in NHWC) with fully coalesced 16-byte loads, 8 in flight per
// thread; per-cell dot products are reduced per pixel group with shuffles and
// one shared-memory atomic per group; then decisions + the tile's compaction
// (tile = the strip's cells, row-major) with decoupled look-back.
// ---------------------------------------------------------------------------
template <typename T, int UNROLL>
__global__ void __launch_bounds__(256) masker_strip_kernel(
    const T* __restrict__ x, int ld, int n, int h, int w, int c, int win, int cells_h, int cells_w,
    const float* __restrict__ wdiff, float bias, float inv_area, uint8_t* __restrict__ coarse,
    float* __restrict__ dots, int dots_stride, int* __restrict__ list, int* __restrict__ count,
    ScanState* st, int num_tiles) {
  extern __shared__ float s_w[];  // c floats, then cells_w sums
  float* s_sum = s_w + c;
  __shared__ int s_tile, s_excl, s_rel, s_wc[8];
  if (threadIdx.x == 0) s_tile = (int)atomicAdd(&st->tile_ctr, 1u);
  for (int i = threadIdx.x; i < c; i += blockDim.x) s_w[i] = wdiff[i];
  for (int i = threadIdx.x; i < cells_w; i += blockDim.x) s_sum[i] = 0.f;
  __syncthreads();
  const int tile = s_tile;  // = n * cells_h + ci
  const int ni = tile / cells_h, ci = tile - (tile / cells_h) * cells_h;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cpp = c >> 3;                       // 8-channel chunks per pixel (power of 2)
  const int grp = cpp < 32 ? cpp : 32;          // lanes sharing one pixel
  const int lcpp = __ffs(cpp) - 1;               // cpp is a power of two
  const int row_chunks = w * cpp;
  const int total = row_chunks * win;            // chunks in the strip
  const T* base = x + (size_t)(ni * h + ci * win) * w * ld;
  for (int q0 = threadIdx.x; q0 < total; q0 += blockDim.x * UNROLL) {
    float part[UNROLL];
    int cell_of[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int q = q0 + u * blockDim.x;
      part[u] = 0.f;
      cell_of[u] = -1;
      if (q < total) {
        const int pxl = q >> lcpp;               // pixel index within the strip
        const int ch = (q & (cpp - 1)) << 3;
        const int r = pxl / w;
        const int px = pxl - r * w;
        part[u] = dot8<T>(base + ((size_t)r * w + px) * ld + ch, s_w + ch);
        cell_of[u] = px / win;
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      float v = part[u];
      for (int o = 1; o < grp; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((lane & (grp - 1)) == 0 && cell_of[u] >= 0) atomicAdd(&s_sum[cell_of[u]], v);
    }
  }
  __syncthreads();
  // decisions and compaction of this strip's cells_w cells (<= 256)
  const int cell0 = tile * cells_w;
  bool mine = false;
  if (threadIdx.x < cells_w) {
    const float d = s_sum[threadIdx.x];
    mine = d * inv_area + bias >= 0.f;
    coarse[cell0 + threadIdx.x] = mine ? 1 : 0;
    if (dots) {  // same layout as the split partials: [cell][split], extra splits zero
      float* dp = dots + (size_t)(cell0 + threadIdx.x) * dots_stride;
      dp[0] = d;
      for (int k = 1; k < dots_stride; ++k) dp[k] = 0.f;
    }
  }
  const unsigned bal = __ballot_sync(0xffffffffu, mine);
  if (lane == 0) s_wc[warp] = __popc(bal);
  __syncthreads();
  if (warp == 0) {
    const int v = lane < 8 ? s_wc[lane] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      const int u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane < 8) s_wc[lane] = incl - v;
    const int agg = __shfl_sync(0xffffffffu, incl, 7);
    const int excl = warp_lookback(st, tile, agg, lane);
    if (lane == 0) {
      s_excl = excl;
      if (tile == num_tiles - 1) *count = excl + agg;
    }
  }
  __syncthreads();
  if (mine) list[s_excl + s_wc[warp] + __popc(bal & ((1u << lane) - 1u))] = cell0 + threadIdx.x;
  scan_state_release(st, num_tiles, &s_rel);
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
size_t scan_state_bytes(int total) {
  const int tiles = total + 2;  // strip-masker tiles may hold a single item (layer masker)
  return sizeof(ScanState) + sizeof(unsigned long long) * (tiles > 0 ? tiles : 1);
}

template <class Flag>
static cudaError_t launch_compact(const Flag& f, int total, int* list, int* count, void* scan,
                                  cudaStream_t stream) {
  const int tiles = (total + CT_TILE - 1) / CT_TILE;
  if (tiles == 0) return cudaMemsetAsync(count, 0, sizeof(int), stream);
  launch_k(compact_kernel<Flag>, dim3(tiles), dim3(CT_THREADS), 0, stream, f, total, list, count,
                                                         reinterpret_cast<ScanState*>(scan), tiles);
  return cudaGetLastError();
}

int masker_splits(int win, int c, int* chunks_per_split) {
  const int cell_chunks = win * win * (c / 8);
  const int budget = 1024;  // 16 KiB of x per warp work item
  const int splits = (cell_chunks + budget - 1) / budget;
  *chunks_per_split = (cell_chunks + splits - 1) / splits;
  return splits;
}

cudaError_t launch_spatial_masker(const void* x, int x_f32, int ld, int n, int h, int w, int c,
                                  int s, int stride, const float* wdiff, float bias,
                                  uint8_t* coarse, int* list, int* count, float* partial,
                                  void* scan, cudaStream_t stream, const uint8_t* prev_coarse,
                                  float* dn) {
  const int win = s * stride;
  const int cells_h = h / win, cells_w = w / win;
  int cps = 0;
  const int splits = masker_splits(win, c, &cps);
  const int total = n * cells_h * cells_w;
  const int cpp = c / 8;
  const bool pow2 = cpp > 0 && (cpp & (cpp - 1)) == 0;
  // experimental (slower and not race-free yet): LAUD_MASKER_STRIP=1
  if (!dn && total > 0 && pow2 && cells_w <= 256 && getenv("LAUD_MASKER_STRIP")) {
    // streaming strip masker: decisions + compaction in one launch
    const int tiles = n * cells_h;
    const float inv_area = 1.0f / (float)(win * win);
    const size_t sm = (size_t)(c + cells_w) * sizeof(float);
    if (x_f32)
      masker_strip_kernel<float, 4><<<tiles, 256, sm, stream>>>(
          reinterpret_cast<const float*>(x), ld, n, h, w, c, win, cells_h, cells_w, wdiff, bias,
          inv_area, coarse, partial, splits, list, count, reinterpret_cast<ScanState*>(scan), tiles);
    else
      masker_strip_kernel<__nv_bfloat16, 8><<<tiles, 256, sm, stream>>>(
          reinterpret_cast<const __nv_bfloat16*>(x), ld, n, h, w, c, win, cells_h, cells_w,
          wdiff, bias, inv_area, coarse, partial, splits, list, count,
          reinterpret_cast<ScanState*>(scan), tiles);
    return cudaGetLastError();
  }
  static const int fused_max = [] {
    const char* e = getenv("LAUD_MASKER_FUSED_MAX");
    return e ? atoi(e) : 4096;
  }();
  if (splits == 1 && total > 0 && total <= fused_max && !dn) {  // small grids: one launch wins
    // one pass: dots + decisions + compaction; ~2 waves of CTAs over the SMs
    // one cell per warp: as many resident warps (bytes in flight) as the SMs hold
    // warps per cell: as many as keep the grid within one wave of resident
    // CTAs (8 per SM) — small batches are latency-bound, so a cell's bytes are
    // spread over more warps (batch 1 R101: masker 12.3 -> 8.2 us per block)
    static const int wpc_env = [] {
      const char* e = getenv("LAUD_MASKER_WPC");  // override: 1, 2, 4 or 8
      return e ? atoi(e) : 0;
    }();
    static const int num_sms = [] {
      int dev = 0, v = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
      return v;
    }();
    int wpc = 1;
    if (wpc_env == 1 || wpc_env == 2 || wpc_env == 4 || wpc_env == 8) {
      wpc = wpc_env;
    } else {
      while (wpc < 8 && (long long)total * wpc * 2 / 8 <= 8LL * num_sms) wpc *= 2;
    }
    const int tc = 8 / wpc;
    const int tiles = (total + tc - 1) / tc;
    const float inv_area = 1.0f / (float)(win * win);
    if (x_f32)
      launch_k(masker_fused_kernel<float>, dim3(tiles), dim3(256), c * sizeof(float), stream, 
          reinterpret_cast<const float*>(x), ld, n, h, w, c, win, cells_h, cells_w, wdiff, bias,
          inv_area, tc, coarse, partial, list, count, reinterpret_cast<ScanState*>(scan), tiles);
    else
      launch_k(masker_fused_kernel<__nv_bfloat16>, dim3(tiles), dim3(256), c * sizeof(float), stream, 
          reinterpret_cast<const __nv_bfloat16*>(x), ld, n, h, w, c, win, cells_h, cells_w, wdiff,
          bias, inv_area, tc, coarse, partial, list, count, reinterpret_cast<ScanState*>(scan), tiles);
    return cudaGetLastError();
  }
  const long long items = (long long)total * splits;
  const int blocks = (int)((items + 7) / 8);
  const int cell_chunks = win * win * (c / 8);
  // layer masker (one cell per image, contiguous rows): the register-weight kernel
  static const int contig_env = [] {
    const char* e = getenv("LAUD_CELL_DOT_CONTIG");
    return e ? atoi(e) : 1;
  }();
  const int P = c / 256;
  if (contig_env && !x_f32 && !dn && cells_h == 1 && cells_w == 1 && win == h && win == w && ld == c &&
      c % 256 == 0 && (P == 1 || P == 2 || P == 4 || P == 8) && splits == (cell_chunks + 1023) / 1024) {
    auto* xb = reinterpret_cast<const __nv_bfloat16*>(x);
    if (P == 1)
      launch_k(cell_dot_contig_kernel<1>, dim3(blocks), dim3(256), 0, stream, xb, cell_chunks, wdiff, splits, partial, items);
    else if (P == 2)
      launch_k(cell_dot_contig_kernel<2>, dim3(blocks), dim3(256), 0, stream, xb, cell_chunks, wdiff, splits, partial, items);
    else if (P == 4)
      launch_k(cell_dot_contig_kernel<4>, dim3(blocks), dim3(256), 0, stream, xb, cell_chunks, wdiff, splits, partial, items);
    else
      launch_k(cell_dot_contig_kernel<8>, dim3(blocks), dim3(256), 0, stream, xb, cell_chunks, wdiff, splits, partial, items);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    MaskerFlag f{partial, splits, 1.0f / (float)(win * win), bias, coarse};
    return launch_compact(f, total, list, count, scan, stream);
  }
  if (false && !x_f32 && splits == 1 && cell_chunks <= 512) {  // measured slower (occupancy)
    auto* xb = reinterpret_cast<const __nv_bfloat16*>(x);
    const size_t sm = c * sizeof(float);
    if (cell_chunks <= 128)
      cell_dot_unrolled_kernel<4><<<blocks, 256, sm, stream>>>(xb, ld, n, h, w, c, win, cells_h,
                                                               cells_w, wdiff, partial);
    else if (cell_chunks <= 256)
      cell_dot_unrolled_kernel<8><<<blocks, 256, sm, stream>>>(xb, ld, n, h, w, c, win, cells_h,
                                                               cells_w, wdiff, partial);
    else
      cell_dot_unrolled_kernel<16><<<blocks, 256, sm, stream>>>(xb, ld, n, h, w, c, win, cells_h,
                                                                cells_w, wdiff, partial);
  } else if (x_f32)
    launch_k(cell_dot_kernel<float>, dim3(blocks), dim3(256), c * sizeof(float), stream, 
        reinterpret_cast<const float*>(x), ld, n, h, w, c, win, cells_h, cells_w, wdiff, splits,
        cps, partial, prev_coarse, dn);
  else
    launch_k(cell_dot_kernel<__nv_bfloat16>, dim3(blocks), dim3(256), c * sizeof(float), stream, 
        reinterpret_cast<const __nv_bfloat16*>(x), ld, n, h, w, c, win, cells_h, cells_w, wdiff,
        splits, cps, partial, prev_coarse, dn);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  MaskerFlag f{partial, splits, 1.0f / (float)(win * win), bias, coarse};
  return launch_compact(f, total, list, count, scan, stream);
}

// Decisions + active-cell list from the per-pixel masker dots conv1's fused
// readers stored (dots [n][h][w] on conv1's input grid, win = S * stride).
cudaError_t launch_masker_decide(const float* pixel_dots, int n, int h, int w, int win, float bias,
                                 uint8_t* coarse, int* list, int* count, void* scan, cudaStream_t stream) {
  const int cells_h = h / win, cells_w = w / win;
  PixelWindowFlag f{pixel_dots, h, w, win, cells_h, cells_w, 1.0f / (float)(win * win), bias, coarse};
  return launch_compact(f, n * cells_h * cells_w, list, count, scan, stream);
}

cudaError_t launch_list_from_mask(const uint8_t* coarse, int total, int* list, int* count,
                                  void* scan, cudaStream_t stream) {
  GivenFlag f{coarse};
  return launch_compact(f, total, list, count, scan, stream);
}

cudaError_t launch_dilate_pixels(const uint8_t* coarse, int n, int h, int w, int s, int stride,
                                 int cells_h, int cells_w, int radius, int* list, int* count,
                                 void* scan, cudaStream_t stream) {
  DilateFlag f{coarse, h, w, s, stride, cells_h, cells_w, radius};
  return launch_compact(f, n * h * w, list, count, scan, stream);
}

}  // namespace laud
