#pragma once
// Implicit-GEMM convolution engine on tcgen05 / TMEM / TMA (sm_100a).
//
// Persistent, warp-specialised kernel (704 threads, 1 CTA per SM; PAIR: one
// 2-CTA cluster per TPC issuing cta_group::2 MMAs):
//   warps 0-3   A producer: one TMA box (contiguous rows), 4D patch boxes or
//               tile::gather4 (4 arbitrary rows per op, OOB -> zero halo) per
//               (tap, 64-channel block), 128B-swizzled K-major; warps 1-3 also
//               run the fused masker dots for conv1 (AM_TILE_DOT);
//   warp 4      B producer: one TMA tile of the packed weights per stage;
//   warp 5      MMA issuer: 4 x tcgen05.mma (128 x BN x 16) per stage into
//               double-buffered TMEM accumulators (four for BN <= 128);
//   warps 6-21  epilogue: tcgen05.ld -> bias (smem cache) [+ residual] [+ ReLU]
//               -> bf16 rows staged in smem -> coalesced 16-byte row stores to
//               the destination pixel (scatter) or compact row; BN <= 128 runs
//               two groups of 8 warps on alternate tiles.
// Row enumeration (dense grid / active-patch list / pixel list) and the
// device-side row count make the same kernel serve the gather-conv1, patch
// conv2 (3x3 halo via zero-filled gathers) and conv3+scatter-add steps of
// LAUDNet's schedule (reference semantics: `reference.py:378-403`).  Kernels
// are instantiated per A mode and epilogue mode so each launch fetches only
// its own code path.
#include <cuda.h>
#include <cuda_runtime.h>

#include "laud_conv.cuh"
#include "laud_launch.cuh"
#include "laud_ptx.cuh"
#include "laud_rows.cuh"

namespace laud {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int A_STAGE_BYTES = BM * BK * 2;  // 16 KiB
#ifndef LAUD_EPI_WARPS
#define LAUD_EPI_WARPS 16
#endif
constexpr int WARP_TMA = 4;
constexpr int WARP_MMA = 5;
constexpr int FIRST_EPI = 6;
constexpr int NUM_EPI_WARPS = LAUD_EPI_WARPS;  // warps 6 .. 6 + NUM_EPI_WARPS - 1
constexpr int NUM_THREADS = (FIRST_EPI + NUM_EPI_WARPS) * 32;
// floats of the per-kernel smem vector cache (bias; + masker weights): the
// epilogue vector region, 3 x 64 floats per epilogue warp for every tile width
constexpr int VEC_CACHE_FLOATS = NUM_EPI_WARPS * 3 * 64;

// Raw list entry row m depends on (fetched early; map_row_raw resolves it).
__device__ __forceinline__ int row_fetch(const ConvParams& p, int m) {
  if (p.list == nullptr || p.sample_rows > 0 || p.row_mode == ROWS_DENSE) return 0;
  int idx, lim;
  if (p.row_mode == ROWS_PATCH) {
    const int s2 = p.patch_h * p.patch_w;
    idx = m / s2;
    lim = (p.rows_max - 1) / s2;
  } else {
    idx = m;
    lim = p.rows_max - 1;
  }
  idx = min(idx, lim);  // unconditional: consumed later
  return p.row_mode == ROWS_PATCH ? list_cell(p, idx) : __ldg(p.list + idx);
}
__device__ __forceinline__ bool map_row_raw(const ConvParams& p, int m, int nvalid, int raw, RowPos& o,
                                            bool& first_patch) {
  first_patch = false;
  if (m >= nvalid) return false;
  const int hw = p.out_h * p.out_w;
  if (p.row_mode == ROWS_PATCH) {
    const int s2 = p.patch_h * p.patch_w;
    const int pi = m / s2;
    const int l = m - pi * s2;
    const int cpi = p.cells_h * p.cells_w;
    o.n = raw / cpi;
    const int c = raw - o.n * cpi;
    const int ci = c / p.cells_w;
    const int cj = c - ci * p.cells_w;
    const int ly = l / p.patch_w;
    o.y = ci * p.patch_h + ly;
    o.x = cj * p.patch_w + (l - ly * p.patch_w);
    o.pix = (o.n * p.out_h + o.y) * p.out_w + o.x;
    first_patch = (pi == 0);
    return true;
  }
  int pix;
  if (p.sample_rows > 0) {
    const int smp = m / p.sample_rows;
    const int loc = m - smp * p.sample_rows;
    if (loc >= hw) return false;
    pix = smp * hw + loc;
  } else {
    pix = (p.row_mode == ROWS_PIXEL) ? raw : m;
  }
  o.pix = pix;
  o.n = pix / hw;
  const int r = pix - o.n * hw;
  o.y = r / p.out_w;
  o.x = r - o.y * p.out_w;
  return true;
}

// Per-tile schedule shared by every warp role (all roles skip the same tiles).
struct TileInfo {
  int m0, n0, sample, kpt, num_kb, kc;
  int kb_lo, kb_hi;  // this CTA's k-blocks (all; or its slice under cluster split-K)
  int c_lo;  // first input channel of the tile's K window (grouped convs)
  bool skip;
};
template <int BN, bool PAIR = false>
__device__ __forceinline__ TileInfo tile_info(const ConvParams& p, int t, int n_tiles, int rank = 0) {
  TileInfo ti;
  // a pair tile is 256 rows: CTA `rank` of the pair owns rows 128*rank ..
  ti.m0 = (t / n_tiles) * (PAIR ? 2 * BM : BM) + (PAIR ? rank * BM : 0);
  ti.n0 = (t % n_tiles) * BN;
  ti.sample = p.sample_rows > 0 ? ti.m0 / p.sample_rows : 0;
  ti.kc = p.chan_count ? __ldg(p.chan_count + ti.sample) : 0;
  ti.skip = p.chan_count && p.n_dyn && ti.n0 >= ti.kc;
  ti.kpt = (p.chan_count && p.k_dyn) ? (ti.kc + BK - 1) / BK : p.kpad / BK;
  ti.c_lo = 0;
  if (p.groups > 1) {  // the input channels of the groups this N tile touches
    const int g0 = ti.n0 / p.gw_out;
    const int g1 = min(p.groups, (min(ti.n0 + BN, p.n_out) + p.gw_out - 1) / p.gw_out);
    ti.c_lo = g0 * p.gw_in;
    ti.kpt = ((g1 - g0) * p.gw_in + BK - 1) / BK;
  }
  ti.num_kb = p.ksize * p.ksize * ti.kpt;
  ti.kb_lo = 0;
  ti.kb_hi = ti.num_kb;
  if (BN == 64 && !PAIR && p.ksplit > 1) {  // small grids: CTA ks of the cluster takes K slice ks
    const int ks = (int)cluster_ctarank();
    ti.kb_lo = ks * ti.num_kb / p.ksplit;
    ti.kb_hi = (ks + 1) * ti.num_kb / p.ksplit;
  }
  return ti;
}

template <int BN, int STAGES, int NSTG, bool PAIR = false>
struct Smem {
  static constexpr int B_STAGE_BYTES = (PAIR ? BN / 2 : BN) * BK * 2;  // this CTA's B rows
  static constexpr int A_OFF = 0;
  static constexpr int B_OFF = STAGES * A_STAGE_BYTES;
  // narrow tiles (BN <= 128, NSTG staging buffers): the epilogue warps form
  // NSTG groups that finish consecutive tiles concurrently (each group its own
  // staging buffer and TMEM accumulators), so per-tile epilogue latency overlaps
  // (BN = 64: four groups of 4 warps, one per staging buffer — small-K convs
  // are bound by the per-tile epilogue latency, so more tiles finish at once)
  static constexpr int EG = (BN <= 128 && NSTG >= 2 && !PAIR) ? NSTG : 1;
  static constexpr int NACC = 2 * EG;  // TMEM accumulators in flight
  static constexpr int EW_COLS0 = BN / (NUM_EPI_WARPS / EG / 4);
  // staging rows: 16-byte chunks XOR-swizzled by row when a warp's slice is 8
  // chunks wide (conflict-free row-per-lane and row-major access, no padding);
  // narrower slices are padded instead
  static constexpr bool STG_SWZ = EW_COLS0 == 64;
  static constexpr int STG_ROW = STG_SWZ ? BN * 2 : BN * 2 + 16;
  static constexpr int STG_OFF = B_OFF + STAGES * B_STAGE_BYTES;
  static constexpr int STG_BUF = BM * STG_ROW;  // one staging buffer
  static constexpr int VEC_OFF = STG_OFF + NSTG * STG_BUF;  // per-warp scale/bias slices
  static constexpr int EW_COLS = EW_COLS0;  // columns per epilogue warp
  static constexpr int VEC_BYTES = NUM_EPI_WARPS * 3 * EW_COLS * 4;  // scale, bias, next wdiff
  static_assert(VEC_BYTES / 4 >= VEC_CACHE_FLOATS, "vector cache size");
  static constexpr int BAR_OFF = VEC_OFF + VEC_BYTES;
  static constexpr int NUM_BARS = 2 * STAGES + 2 * NACC;
  static constexpr int TMEM_SLOT_OFF = BAR_OFF + NUM_BARS * 8;
  static constexpr int BIDX_OFF = TMEM_SLOT_OFF + 16;  // gathered-B row indices of the current tile
  static constexpr int BIDX_INTS = BN > BK ? BN : BK;
  static constexpr int BYTES = BIDX_OFF + BIDX_INTS * 4;
  static constexpr int ALLOC = BYTES + 1024;  // manual 1 KiB alignment
  static constexpr uint32_t TMEM_COLS = NACC * BN;
};

// A-operand producer compiled into an instantiation (the kernel carries every
// role; keeping only the launch's A path shrinks the code the warps fetch)
enum AMode { AM_TILE = 0, AM_BOX = 1, AM_G4 = 2, AM_ANY = 3, AM_TILE_DOT = 4 };
// epilogue compiled in: EP_PLAIN = bf16 out, bias from the smem cache, optional
// residual / ReLU / per-sample channel mask, every warp slice full; EP_ANY = all
// _RES: with the residual add; _RELU: ReLU on every row (no per-cell ReLU mask)
enum EpMode { EP_PLAIN = 0, EP_ANY = 1, EP_PLAIN_RES = 2, EP_PLAIN_RELU = 4, EP_PLAIN_RES_RELU = 6 };

template <int BN, int STAGES, int NSTG, bool PAIR, int AM, int EP>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    conv_gemm_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                     const __grid_constant__ CUtensorMap tmap_o, const ConvParams p) {
  using L = Smem<BN, STAGES, NSTG, PAIR>;
  // PAIR: a cluster of 2 CTAs on one TPC runs M = 256 tiles with
  // tcgen05.mma.cta_group::2 issued by the leader (rank 0); each CTA loads
  // its 128 A rows and half of B, so per-SM operand traffic per MMA halves.
  const int rank = PAIR ? (int)cluster_ctarank() : 0;
  // cluster split-K (small grids, plain epilogues): the KS CTAs of a cluster
  // share one tile, each a slice of its k-blocks; fp32 partials are reduced
  // through distributed shared memory after the role loops
  // (64-wide tiles only: the small-grid tile width; wider instantiations carry no split code)
  constexpr bool kSplitOK = BN == 64 && !PAIR && EP != EP_ANY && BM * (BN + 4) * 4 <= L::STG_OFF;
  const int KS = (kSplitOK && p.ksplit > 1) ? p.ksplit : 1;
  const int t_begin = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x / KS;
  const int t_step = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x / KS;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  const uint32_t base_u32 = (raw_u32 + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_u32 - raw_u32);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + L::BAR_OFF);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* acc_full = bars + 2 * STAGES;
  uint64_t* acc_empty = bars + 2 * STAGES + L::NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + L::TMEM_SLOT_OFF);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  unsigned long long* const trc = (p.trace && blockIdx.x == 0) ? p.trace : nullptr;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      // arrivals: A expect_tx (TMA) or 128 cp.async threads, + B expect_tx or 32 cp.async lanes
      // (fused masker: one thread issues A and B together, warps 0-3 all read)
      mbar_init(&full[s], (AM == AM_TILE_DOT && p.adot_out) ? 1 : (p.a_tma ? 1 : 128) + (p.b_gather != B_BOX ? 32 : 1));
      mbar_init(&empty[s], p.adot_out ? 2 : 1);  // + the fused masker readers
    }
    for (int a = 0; a < L::NACC; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], (PAIR ? 2 : 1) * NUM_EPI_WARPS / L::EG);  // one arrive per group warp
    }
    fence_barrier_init();
  }
  if (warp == WARP_TMA && lane == 0) {
    if (p.b_gather == B_BOX) tma_prefetch_desc(&tmap_b);
    if (p.a_tma) tma_prefetch_desc(&tmap_a);
  }
  if (warp == WARP_MMA) {
    if constexpr (PAIR)
      tmem_alloc_pair<L::TMEM_COLS>(tmem_slot);
    else
      tmem_alloc<L::TMEM_COLS>(tmem_slot);
  }
  tc_fence_before();
  if constexpr (PAIR)
    cluster_sync();  // barrier inits visible cluster-wide before any remote arrive
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // TMA completions go to the (leader's) full barrier; expect_tx only on the leader
  auto full_tx = [&](int stage) -> uint32_t {
    return PAIR ? mapa_shared(smem_u32(&full[stage]), 0) : smem_u32(&full[stage]);
  };
  constexpr uint32_t XMUL = PAIR ? 2u : 1u;  // the leader expects both CTAs' bytes
  const bool leader = rank == 0;
  // PDL: everything above overlaps the previous kernel's tail; from here on the
  // row counts / activations it produced are read
  pdl_wait();
  pdl_trigger();
  const int nvalid = rows_valid(p);
  // K order: for each 64-channel block, the k x k taps (the order of the halo
  // patch conv, patch_conv.cu, so the sparse and dense conv2 sum identically)
  const int taps = p.ksize * p.ksize;
  const int n_tiles = (p.n_out + BN - 1) / BN;
  const int m_tiles = (nvalid + (PAIR ? 2 * BM : BM) - 1) / (PAIR ? 2 * BM : BM);
  const int tiles = m_tiles * n_tiles;

  if (t_begin >= tiles) {
    // no tile for this CTA (uniform across the pair): straight to teardown
  } else if (warp < 4) {
    // ------------------------------------------------------------ A producers
    const int tid = threadIdx.x;
    uint32_t it = 0;
    constexpr bool kTile = AM == AM_TILE || AM == AM_TILE_DOT || AM == AM_ANY;
    constexpr bool kDot = AM == AM_TILE_DOT || AM == AM_ANY;
    constexpr bool kBox = AM == AM_BOX || AM == AM_ANY;
    constexpr bool kG4 = AM == AM_G4 || AM == AM_ANY;
    // AM_TILE_DOT: the B-producer thread issues the A boxes too and warps 0-3
    // (128 threads, one row each) are all masker readers
    constexpr int NRD = AM == AM_TILE_DOT ? 128 : 96;
    if (kDot && p.a_tile && p.adot_out && (AM == AM_TILE_DOT || warp >= 1)) {
      // fused masker readers: every A stage, once landed, is also read here —
      // dot of each row with the masker weights W0 - W1 (`reference.py:244-253`)
      // — and released with a second arrive
      const int mt = AM == AM_TILE_DOT ? tid : tid - 32;  // rows mt (and mt + 96 with 96 readers)
      const int ra = mt, rb = mt + NRD;
      // plain-epilogue kernels only use the bias part of the vector region: the
      // masker weights live at its top for the whole kernel (host checks the fit)
      float* const wsm = reinterpret_cast<float*>(base + L::VEC_OFF + L::VEC_BYTES) - p.kpad;
      if constexpr (EP != EP_ANY) {
        for (int i = mt; i < p.kpad; i += NRD) wsm[i] = __ldg(p.adot_w + i);
        asm volatile("bar.sync 3, %0;" ::"n"(NRD) : "memory");
      }
      for (int t = t_begin; t < tiles; t += t_step) {
        const TileInfo ti = tile_info<BN, PAIR>(p, t, n_tiles, rank);
        if (ti.skip) continue;
        float aa[4] = {0.f, 0.f, 0.f, 0.f}, ab[4] = {0.f, 0.f, 0.f, 0.f};  // 4-way ILP per row
        const bool dots = ti.n0 == 0;  // every N tile re-reads the rows: dot them once
        for (int kb = ti.kb_lo; kb < ti.kb_hi; ++kb, ++it) {
          const int stage = it % STAGES;
          const uint32_t phase = (it / STAGES) & 1;
          mbar_wait(&full[stage], phase);
          const uint8_t* sA = base + L::A_OFF + stage * A_STAGE_BYTES;
          if (dots) {
            uint4 va[8], vb[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              va[c] = *reinterpret_cast<const uint4*>(sA + ra * 128 + ((c ^ (ra & 7)) << 4));
              vb[c] = (NRD < BM && rb < BM) ? *reinterpret_cast<const uint4*>(sA + rb * 128 + ((c ^ (rb & 7)) << 4))
                                            : make_uint4(0u, 0u, 0u, 0u);
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              float4 w0, w1;
              if constexpr (EP != EP_ANY) {
                w0 = *reinterpret_cast<const float4*>(wsm + kb * BK + c * 8);
                w1 = *reinterpret_cast<const float4*>(wsm + kb * BK + c * 8 + 4);
              } else {
                w0 = __ldg(reinterpret_cast<const float4*>(p.adot_w + kb * BK + c * 8));
                w1 = __ldg(reinterpret_cast<const float4*>(p.adot_w + kb * BK + c * 8 + 4));
              }
              const int k = c & 3;
              float2 f;
              f = unpack_bf16x2(va[c].x); aa[k] = fmaf(f.x, w0.x, aa[k]); aa[k] = fmaf(f.y, w0.y, aa[k]);
              f = unpack_bf16x2(va[c].y); aa[k] = fmaf(f.x, w0.z, aa[k]); aa[k] = fmaf(f.y, w0.w, aa[k]);
              f = unpack_bf16x2(va[c].z); aa[k] = fmaf(f.x, w1.x, aa[k]); aa[k] = fmaf(f.y, w1.y, aa[k]);
              f = unpack_bf16x2(va[c].w); aa[k] = fmaf(f.x, w1.z, aa[k]); aa[k] = fmaf(f.y, w1.w, aa[k]);
              if constexpr (NRD < BM) {
                f = unpack_bf16x2(vb[c].x); ab[k] = fmaf(f.x, w0.x, ab[k]); ab[k] = fmaf(f.y, w0.y, ab[k]);
                f = unpack_bf16x2(vb[c].y); ab[k] = fmaf(f.x, w0.z, ab[k]); ab[k] = fmaf(f.y, w0.w, ab[k]);
                f = unpack_bf16x2(vb[c].z); ab[k] = fmaf(f.x, w1.x, ab[k]); ab[k] = fmaf(f.y, w1.y, ab[k]);
                f = unpack_bf16x2(vb[c].w); ab[k] = fmaf(f.x, w1.z, ab[k]); ab[k] = fmaf(f.y, w1.w, ab[k]);
              }
            }
          }
          asm volatile("bar.sync 3, %0;" ::"n"(NRD) : "memory");
          if (mt == 0) mbar_arrive(&empty[stage]);
        }
        const float acc_a = (aa[0] + aa[1]) + (aa[2] + aa[3]);
        const float acc_b = (ab[0] + ab[1]) + (ab[2] + ab[3]);
        // one dot per row = per pixel of the dense input grid, stored (no
        // atomics): the decision pass sums each cell's window in a fixed
        // row-major order, so decisions are deterministic run to run
        if (dots) {
          if (ti.m0 + ra < nvalid) p.adot_out[ti.m0 + ra] = acc_a;
          if (NRD < BM && rb < BM && ti.m0 + rb < nvalid) p.adot_out[ti.m0 + rb] = acc_b;
        }
      }
    } else if (kTile && p.a_tile) {
      // Contiguous rows (compact / dense 1x1): one 128 x 64 TMA box per stage.
      if (tid == 0) {
        for (int t = t_begin; t < tiles; t += t_step) {
          const TileInfo ti = tile_info<BN, PAIR>(p, t, n_tiles, rank);
          if (ti.skip) continue;
          const int row0 = p.sample_rows > 0
                               ? ti.sample * p.out_h * p.out_w + (ti.m0 - ti.sample * p.sample_rows)
                               : ti.m0;
          for (int kb = ti.kb_lo; kb < ti.kb_hi; ++kb, ++it) {
            const int stage = it % STAGES;
            const uint32_t phase = (it / STAGES) & 1;
            mbar_wait(&empty[stage], phase ^ 1);
            if (trc && it < 4096) trc[TRACE_A + it] = global_ns();
            const uint32_t sA = base_u32 + L::A_OFF + stage * A_STAGE_BYTES;
            if (p.dbg & 8) {
              if (leader) mbar_arrive(&full[stage]);
            } else if constexpr (PAIR) {
              if (leader) mbar_arrive_expect_tx(&full[stage], XMUL * A_STAGE_BYTES);
              tma_load_2d_pair(sA, &tmap_a, full_tx(stage), ti.c_lo + kb * BK, row0);
            } else {
              mbar_arrive_expect_tx(&full[stage], A_STAGE_BYTES);
              tma_load_2d(sA, &tmap_a, &full[stage], ti.c_lo + kb * BK, row0);
            }
          }
        }
      }
    } else if (kBox && p.a_box) {
      // S x S patches: thread i < 128 / S^2 owns patch i of the tile and loads its
      // tap window as one 4D box (S^2 rows x 64 channels, OOB -> zero halo)
      const int s2 = p.patch_h * p.patch_w;
      const int ppt = BM / s2;  // patches per tile
      const int cpi = p.cells_h * p.cells_w;
      for (int t = t_begin; t < tiles; t += t_step) {
        const TileInfo ti = tile_info<BN, PAIR>(p, t, n_tiles, rank);
        if (ti.skip) continue;
        int bn_ = p.batch, by = 0, bx = 0;  // invalid patch -> image index past the end (zeros)
        const int pi = ti.m0 / s2 + tid;
        if (tid < ppt && pi * s2 < nvalid) {
          const int cell = list_cell(p, pi);
          bn_ = cell / cpi;
          const int cr = cell - bn_ * cpi;
          const int ci = cr / p.cells_w, cj = cr - (cr / p.cells_w) * p.cells_w;
          by = ci * p.patch_h * p.stride - p.pad;
          bx = cj * p.patch_w * p.stride - p.pad;
        }
        for (int kb = ti.kb_lo; kb < ti.kb_hi; ++kb, ++it) {
          const int stage = it % STAGES;
          const uint32_t phase = (it / STAGES) & 1;
          mbar_wait(&empty[stage], phase ^ 1);
          if (trc && tid == 0 && it < 4096) trc[TRACE_A + it] = global_ns();
          const int cblk = kb / taps, tap = kb - cblk * taps;  // channel-block-major K order
          const int c0 = ti.c_lo + cblk * BK;
          const int ky = tap / p.ksize;
          const int kx = tap - ky * p.ksize;
          const uint32_t sA = base_u32 + L::A_OFF + stage * A_STAGE_BYTES;
          if (tid == 0) mbar_arrive_expect_tx(&full[stage], A_STAGE_BYTES);
          if (tid < ppt) tma_load_4d(sA + tid * s2 * 128, &tmap_a, &full[stage], c0, bx + kx, by + ky, bn_);
        }
      }
    } else if (kG4 && p.a_tma) {
      // One output row per thread; per (tap, channel block) every 4th lane issues
      // a TMA tile::gather4 of its 4 rows' source pixels (OOB index -> zeros).
      for (int t = t_begin; t < tiles; t += t_step) {
        const TileInfo ti = tile_info<BN, PAIR>(p, t, n_tiles, rank);
        if (ti.skip) continue;
        const int m0 = ti.m0;
        RowPos rp;
        bool fp;
        const bool rv = map_row(p, m0 + tid, nvalid, rp, fp);
        for (int kb = ti.kb_lo; kb < ti.kb_hi; ++kb, ++it) {
          const int stage = it % STAGES;
          const uint32_t phase = (it / STAGES) & 1;
          mbar_wait(&empty[stage], phase ^ 1);
          if (trc && tid == 0 && it < 4096) trc[TRACE_A + it] = global_ns();
          const int cblk = kb / taps, tap = kb - cblk * taps;  // channel-block-major K order
          const int c0 = ti.c_lo + cblk * BK;
          const int ky = tap / p.ksize;
          const int kx = tap - ky * p.ksize;
          int row = p.a_rows;  // out of bounds -> zero fill
          if (rv) {
            if (p.a_compact) {
              row = p.sample_rows > 0 ? rp.pix : m0 + tid;
            } else {
              const int iy = rp.y * p.stride + ky - p.pad;
              const int ix = rp.x * p.stride + kx - p.pad;
              if (iy >= 0 && iy < p.in_h && ix >= 0 && ix < p.in_w)
                row = (rp.n * p.in_h + iy) * p.in_w + ix;
            }
          }
          const int r1 = __shfl_down_sync(0xffffffffu, row, 1);
          const int r2 = __shfl_down_sync(0xffffffffu, row, 2);
          const int r3 = __shfl_down_sync(0xffffffffu, row, 3);
          const uint32_t sA = base_u32 + L::A_OFF + stage * A_STAGE_BYTES;
          if (tid == 0 && leader) mbar_arrive_expect_tx(&full[stage], XMUL * A_STAGE_BYTES);
          if ((lane & 3) == 0) {
            if constexpr (PAIR)
              tma_gather4_pair(sA + tid * 128, &tmap_a, full_tx(stage), c0, row, r1, r2, r3);
            else
              tma_gather4(sA + tid * 128, &tmap_a, &full[stage], c0, row, r1, r2, r3);
          }
        }
      }
    } else if (AM == AM_ANY) {
    const int chunk = tid & 7;
    const int rsub = tid >> 3;
    const __nv_bfloat16* act = reinterpret_cast<const __nv_bfloat16*>(p.act);
    for (int t = t_begin; t < tiles; t += t_step) {
      const TileInfo ti = tile_info<BN, PAIR>(p, t, n_tiles, rank);
      if (ti.skip) continue;
      const int m0 = ti.m0;
      RowPos rp[8];
      bool rv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        bool fp;
        rv[i] = map_row(p, m0 + rsub + 16 * i, nvalid, rp[i], fp);
      }
      for (int kb = ti.kb_lo; kb < ti.kb_hi; ++kb, ++it) {
        const int stage = it % STAGES;
        const uint32_t phase = (it / STAGES) & 1;
        mbar_wait(&empty[stage], phase ^ 1);
        const int cblk = kb / taps, tap = kb - cblk * taps;
        const int ch = ti.c_lo + cblk * BK + chunk * 8;
        const int ky = tap / p.ksize;
        const int kx = tap - ky * p.ksize;
        const bool chv = ch < p.in_c;
        const uint32_t sA = base_u32 + L::A_OFF + stage * A_STAGE_BYTES;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int r = rsub + 16 * i;
          const uint32_t dst = sA + r * 128 + ((chunk ^ (r & 7)) << 4);
          bool v = rv[i] && chv;
          const __nv_bfloat16* src = act;
          if (p.a_compact) {
            src = act + (size_t)(p.sample_rows > 0 ? rp[i].pix : m0 + r) * p.in_ld + ch;
          } else {
            const int iy = rp[i].y * p.stride + ky - p.pad;
            const int ix = rp[i].x * p.stride + kx - p.pad;
            v = v && iy >= 0 && iy < p.in_h && ix >= 0 && ix < p.in_w;
            src = act + ((size_t)(rp[i].n * p.in_h + iy) * p.in_w + ix) * p.in_ld + ch;
          }
          cp_async_16(dst, v ? (const void*)src : (const void*)act, v ? 16u : 0u);
        }
        cp_async_mbar_arrive_noinc(&full[stage]);
      }
    }
    }
  } else if (warp == WARP_TMA) {
    // ------------------------------------------------------------ B producer (TMA)
    if (p.b_gather != B_BOX) {
      // per-sample weights gathered in-kernel (channel skipping): the warp's 32
      // lanes cp.async the tile's 16-byte chunks into the 128B-swizzled stage
      // (a TMA gather4 per 4 rows measured ~8x slower per byte here); indices
      // past the sample's k_n zero-fill.  The tile's row indices sit in smem.
      int* const bidx = reinterpret_cast<int*>(base + L::BIDX_OFF);
      const __nv_bfloat16* const wsrc = reinterpret_cast<const __nv_bfloat16*>(p.weight_g);
      uint32_t it = 0;
      for (int t = t_begin; t < tiles; t += t_step) {
        const TileInfo ti = tile_info<BN, PAIR>(p, t, n_tiles, rank);
        if (ti.skip) continue;
        const int* idx = p.b_index + (size_t)ti.sample * p.b_index_ld;
        const bool gn = p.b_gather == B_GATHER_N;
        for (int kb = ti.kb_lo; kb < ti.kb_hi; ++kb, ++it) {
          const int stage = it % STAGES;
          const uint32_t phase = (it / STAGES) & 1;
          if (gn ? kb == ti.kb_lo : true) {
            // N gather: the tile's BN rows once per tile; K gather: this k-block's 64 K rows
            __syncwarp();
            const int cnt = gn ? BN : BK, off = gn ? ti.n0 : kb * BK;
            for (int j = lane; j < cnt; j += 32) bidx[j] = off + j < ti.kc ? __ldg(idx + off + j) : -1;
            __syncwarp();
          }
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t dst = base_u32 + L::B_OFF + stage * L::B_STAGE_BYTES;
          if (gn) {
            // K-major [BN rows][64]: row r = weight row bidx[r], 128 B at the k-block's K offset
            const int cblk = kb / taps, tap = kb - cblk * taps;
            const int kcoord = tap * p.kpad + cblk * BK;
#pragma unroll 4
            for (int i = lane; i < BN * 8; i += 32) {
              const int r = i >> 3, c = i & 7;
              const int row = bidx[r];
              const __nv_bfloat16* src = wsrc + (size_t)(row < 0 ? 0 : row) * p.b_ld + kcoord + c * 8;
              cp_async_16(dst + r * 128 + ((c ^ (r & 7)) << 4), src, row < 0 ? 0u : 16u);
            }
          } else {
            // MN-major: BN/64 panels of [64 K rows][64 N] (SW128, 8 KiB each); K row k
            // = transposed-weight row bidx[k], columns n0 + 64 pn ..
#pragma unroll 4
            for (int i = lane; i < BK * (BN / 8); i += 32) {
              const int k = i / (BN / 8), cc = i - k * (BN / 8);
              const int pn = cc >> 3, c = cc & 7;
              const int row = bidx[k];
              const __nv_bfloat16* src = wsrc + (size_t)(row < 0 ? 0 : row) * p.b_ld + ti.n0 + cc * 8;
              cp_async_16(dst + pn * 8192 + k * 128 + ((c ^ (k & 7)) << 4), src, row < 0 ? 0u : 16u);
            }
          }
          cp_async_mbar_arrive_noinc(&full[stage]);
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (lane == 0) {
      uint32_t it = 0;
      for (int t = t_begin; t < tiles; t += t_step) {
        const TileInfo ti = tile_info<BN, PAIR>(p, t, n_tiles, rank);
        if (ti.skip) continue;
        for (int kb = ti.kb_lo; kb < ti.kb_hi; ++kb, ++it) {
          const int stage = it % STAGES;
          const uint32_t phase = (it / STAGES) & 1;
          mbar_wait(&empty[stage], phase ^ 1);
          if (trc && it < 4096) trc[TRACE_B + it] = global_ns();
          if (p.dbg & 16) {
            if (leader) mbar_arrive(&full[stage]);
            continue;
          }
          const int cblk = kb / taps, tap = kb - cblk * taps;
          const int kcoord = tap * p.kpad + ti.c_lo + cblk * BK;  // per-tap stride kpad
          const uint32_t dst = base_u32 + L::B_OFF + stage * L::B_STAGE_BYTES;
          if (AM == AM_TILE_DOT && p.adot_out) {
            // fused masker: this thread issues the stage's A box too (warps 0-3 read it)
            mbar_arrive_expect_tx(&full[stage], A_STAGE_BYTES + L::B_STAGE_BYTES);
            tma_load_2d(base_u32 + L::A_OFF + stage * A_STAGE_BYTES, &tmap_a, &full[stage], ti.c_lo + kb * BK,
                        ti.m0);
          } else if (leader) {
            mbar_arrive_expect_tx(&full[stage], XMUL * L::B_STAGE_BYTES);
          }
          if constexpr (PAIR) {  // this CTA's half of the tile's B rows
            tma_load_2d_pair(dst, &tmap_b, full_tx(stage), kcoord, ti.n0 + rank * (BN / 2));
          } else if (p.b_batched) {
            tma_load_3d(dst, &tmap_b, &full[stage], kcoord, ti.n0, ti.sample);
          } else {
            tma_load_2d(dst, &tmap_b, &full[stage], kcoord, ti.n0);
          }
        }
      }
    }
  } else if (warp == WARP_MMA) {
    // ------------------------------------------------------------ MMA issuer
    // (PAIR: the leader issues M = 256 MMAs for both CTAs; the peer's warp idles)
    // B_GATHER_K tiles are MN-major (instruction descriptor bit 16)
    const uint32_t idesc = umma_idesc_bf16(PAIR ? 2 * BM : BM, BN) | (p.b_gather == B_GATHER_K ? (1u << 16) : 0u);
    const bool b_mn = p.b_gather == B_GATHER_K;
    uint32_t it = 0, local = 0;
    for (int t = t_begin; t < tiles && leader; t += t_step) {
      const TileInfo ti = tile_info<BN, PAIR>(p, t, n_tiles, rank);
      if (ti.skip) continue;
      const int acc = local % L::NACC;
      const uint32_t acc_phase = (local / L::NACC) & 1;
      ++local;
      mbar_wait(&acc_empty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t tmem_d = tmem_base + acc * BN;
      for (int kb = ti.kb_lo; kb < ti.kb_hi; ++kb, ++it) {
        const int stage = it % STAGES;
        const uint32_t phase = (it / STAGES) & 1;
        mbar_wait(&full[stage], phase);
        if (trc && lane == 0 && it < 4096) trc[TRACE_MMA + it] = global_ns();
        fence_proxy_async_smem();
        tc_fence_after();
        if (lane == 0 && !(p.dbg & 32)) {
          const uint32_t sA = base_u32 + L::A_OFF + stage * A_STAGE_BYTES;
          const uint32_t sB = base_u32 + L::B_OFF + stage * L::B_STAGE_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            if constexpr (PAIR)
              umma_bf16_pair(tmem_d, umma_sdesc_sw128(sA + k * 32), umma_sdesc_sw128(sB + k * 32), idesc,
                             kb != ti.kb_lo || k != 0);
            else
              umma_bf16(tmem_d, umma_sdesc_sw128(sA + k * 32),
                        b_mn ? umma_sdesc_sw128_mn(sB + k * 2048, 8192) : umma_sdesc_sw128(sB + k * 32), idesc,
                        kb != ti.kb_lo || k != 0);
          }
          if constexpr (PAIR)
            umma_commit_pair(&empty[stage]);  // frees the stage in both CTAs
          else
            umma_commit(&empty[stage]);
        } else if (lane == 0) {
          mbar_arrive(&empty[stage]);
        }
        __syncwarp();
      }
      if (lane == 0) {
        if constexpr (PAIR)
          umma_commit_pair(&acc_full[acc]);
        else
          umma_commit(&acc_full[acc]);
      }
      __syncwarp();
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // NUM_EPI_WARPS warps: warp w reads TMEM lane quadrant q = w % 4 (rows
    // 32q..32q+31; the hardware restricts a warp to its quadrant) and column
    // slice EW_COLS * ((w - FIRST_EPI) / 4) of the tile.  Lane i owns row
    // 32q+i in the math (tcgen05.ld 32x32b: lane = row, registers = columns);
    // rows are staged through shared memory so the residual read and the
    // destination write are coalesced 16-byte-per-lane row segments (a
    // scattered destination row is contiguous in NHWC).  With NSTG = 2 the
    // residual of the next tile is prefetched (cp.async) into the other
    // staging buffer while this tile is finished and stored.
    constexpr int EW_COLS = L::EW_COLS;  // columns per warp
    constexpr int CPR = EW_COLS / 8;     // 16-byte chunks per staged row slice
    constexpr int CH = EW_COLS < 32 ? EW_COLS : 32;  // columns per TMEM load
    const int q = warp & 3;
    const int ew = warp - FIRST_EPI;
    constexpr int GW = NUM_EPI_WARPS / L::EG;  // warps per epilogue group
    const int grp = ew / GW;                     // group: tiles with local % EG == grp
    const int col0 = ((ew % GW) >> 2) * EW_COLS;
    // one staging buffer per group; with one group and two buffers the next
    // tile's residual is prefetched into the other buffer
    constexpr bool kDoubleStage = NSTG == 2 && L::EG == 1;
    // swizzled staging is slice-major: each warp column slice owns BM rows of
    // 128 B (chunk c of row r at c ^ (r & 7): the TMA SWIZZLE_128B layout, so a
    // slice's rows can leave by TMA store boxes); unswizzled: row-major rows
    constexpr int SROW = L::STG_SWZ ? EW_COLS * 2 : L::STG_ROW;
    const int stg_off0 = L::STG_OFF + grp * L::STG_BUF +
                         (L::STG_SWZ ? (col0 / EW_COLS) * BM * SROW + q * 32 * SROW : q * 32 * SROW + col0 * 2);
    // byte offset of 16-byte chunk c of slice row r (relative to stg_off0)
    auto soff = [](int r, int c) { return r * SROW + ((L::STG_SWZ ? (c ^ (r & 7)) : c) << 4); };
    float* const vsc = reinterpret_cast<float*>(base + L::VEC_OFF) + ew * 3 * EW_COLS;
    float* const vbi_w = vsc + EW_COLS;
    float* const vnw = vbi_w + EW_COLS;  // next block's masker weights (masker-conv3 fusion)
    const __nv_bfloat16* resid = reinterpret_cast<const __nv_bfloat16*>(p.resid);
    __nv_bfloat16* outp = reinterpret_cast<__nv_bfloat16*>(p.out);
    const bool staged = !p.out_f32;
    constexpr bool kRes = EP == EP_PLAIN_RES || EP == EP_PLAIN_RES_RELU;
    constexpr bool kReluAll = EP == EP_PLAIN_RELU || EP == EP_PLAIN_RES_RELU;
    const bool pre = (EP != EP_ANY ? kRes : (staged && resid != nullptr)) && KS == 1;  // split-K: resid in the reduction
    const bool has_scale = p.scale != nullptr || p.col_index != nullptr;
    // the common epilogues (bias [+ residual] [+ ReLU]) take a branch-free path
    constexpr bool kPlain = EP != EP_ANY;  // host: plain && cached && full slices
    const bool tma_out = kPlain && L::STG_SWZ && p.tma_out != 0;
    const bool plain = kPlain || (staged && !has_scale && !p.ymask_coarse && !p.mdot_w);
    // the whole bias vector lives in smem for the kernel when it fits (the
    // per-warp vector slices are the fallback for scale / masker-dot / lists)
    const bool cached = kPlain || (!has_scale && !p.mdot_w && (p.n_out + BN - 1) / BN * BN <= L::VEC_BYTES / 4);
    float* const bias_cache = reinterpret_cast<float*>(base + L::VEC_OFF);
    if (cached) {
      // padded to whole tiles: the plain path reads full warp slices (columns
      // past n_out are computed but never stored)
      const int npad = (p.n_out + BN - 1) / BN * BN;
      for (int i = threadIdx.x - FIRST_EPI * 32; i < npad; i += NUM_EPI_WARPS * 32)
        bias_cache[i] = (p.bias && i < p.n_out) ? __ldg(p.bias + i) : 0.f;
      asm volatile("bar.sync 1, %0;" ::"n"(NUM_EPI_WARPS * 32) : "memory");
    }

    // per-row destination of tile t for this lane's row
    struct RowInfo {
      bool valid;
      long long dst;
      RowPos rp;
      bool fp;
    };
    constexpr int MT = PAIR ? 2 * BM : BM;  // rows per (pair) tile
    auto row_raw = [&](int t) { return row_fetch(p, (t / n_tiles) * MT + rank * BM + q * 32 + lane); };
    auto row_info = [&](int t, int raw) {
      RowInfo ri;
      const int m = (t / n_tiles) * MT + rank * BM + q * 32 + lane;
      ri.valid = map_row_raw(p, m, nvalid, raw, ri.rp, ri.fp);
      ri.dst = 0;
      if (ri.valid) {
        if (p.out_mode == OUT_ROW) {
          ri.dst = p.sample_rows > 0 ? ri.rp.pix : m;
        } else {
          int y = ri.rp.y;
          if (p.misplace_first && ri.fp) y = (y + p.patch_h) % p.out_h;
          ri.dst = (long long)(ri.rp.n * p.out_h + y) * p.out_w + ri.rp.x;
        }
      }
      return ri;
    };
    auto prefetch = [&](int t, const RowInfo& ri, int buf) {
      if (tma_out) {  // the buffer's previous TMA store must have read its rows
        bulk_wait_read<0>();
        __syncwarp();
      }
      if (p.dbg & 64) {  // ablation: no residual loads
        asm volatile("cp.async.commit_group;" ::: "memory");
        return;
      }
      const int c_base = (t % n_tiles) * BN + col0;
      const int vchunks = max(0, min(EW_COLS, p.n_out - c_base)) >> 3;
      const uint32_t sbase = base_u32 + stg_off0 + buf * L::STG_BUF;
#pragma unroll 4
      for (int idx = lane; idx < 32 * CPR; idx += 32) {
        const int r = idx / CPR, c = idx % CPR;
        const int rv = __shfl_sync(0xffffffffu, (int)ri.valid, r);
        const long long dr = __shfl_sync(0xffffffffu, ri.dst, r);
        const bool ok = rv && c < vchunks;
        const __nv_bfloat16* src = resid + dr * p.resid_ld + c_base + c * 8;
        cp_async_16(sbase + soff(r, c), ok ? (const void*)src : (const void*)resid,
                    ok ? 16u : 0u);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    auto next_valid = [&](int t) {
      while (t < tiles && tile_info<BN, PAIR>(p, t, n_tiles, rank).skip) t += t_step;
      return t;
    };
    // per-column epilogue vectors of tile t: loads issued a tile ahead (into
    // registers), written to the warp's smem slice once the previous tile's
    // math is done
    constexpr int VPL = (EW_COLS + 31) / 32;  // vector entries per lane
    struct VecPre {
      float sc[VPL], bi[VPL], nw[VPL];
    };
    auto vec_load = [&](int t) {
      VecPre v;
      const TileInfo tv = tile_info<BN, PAIR>(p, t, n_tiles, rank);
      const int cb = tv.n0 + col0;
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        const int i = lane + 32 * u;
        const int c = cb + i;
        int src = c;
        bool live = i < EW_COLS && c < p.n_out;
        if (p.col_index) {  // per-sample channel list: column c holds channel col_index[c]
          live = live && c < tv.kc;
          src = live ? __ldg(p.col_index + (size_t)tv.sample * p.col_index_ld + c) : 0;
        }
        v.sc[u] = (p.scale && live) ? __ldg(p.scale + src) : 1.f;
        v.bi[u] = (p.bias && live) ? __ldg(p.bias + src) : 0.f;
        v.nw[u] = (p.mdot_w && live) ? __ldg(p.mdot_w + c) : 0.f;
      }
      return v;
    };
    auto vec_store = [&](const VecPre& v) {
#pragma unroll
      for (int u = 0; u < VPL; ++u) {
        const int i = lane + 32 * u;
        if (i < EW_COLS) {
          if (has_scale) vsc[i] = v.sc[u];
          vbi_w[i] = v.bi[u];
          if (p.mdot_w) vnw[i] = v.nw[u];
        }
      }
    };
    uint32_t local = 0;
    int t = next_valid(t_begin);
    for (int g = 0; g < grp && t < tiles; ++g) t = next_valid(t + t_step);  // group g starts at the g-th tile
    local = grp;
    RowInfo cur;
    if (t < tiles) {
      cur = row_info(t, row_raw(t));
      if (pre) prefetch(t, cur, 0);
      if (!cached) vec_store(vec_load(t));
      __syncwarp();
    }
    for (; t < tiles; local += L::EG) {
      const TileInfo ti = tile_info<BN, PAIR>(p, t, n_tiles, rank);
      const int acc = local % L::NACC;
      const uint32_t acc_phase = (local / L::NACC) & 1;
      const int buf = kDoubleStage ? (local & 1) : 0;
      uint8_t* stg = base + stg_off0 + buf * L::STG_BUF;
      const int c_base = ti.n0 + col0;                        // first output channel of this warp
      const int nch = max(0, min(EW_COLS, p.n_out - c_base));  // valid channels (multiple of 8)
      const int vchunks = nch >> 3;
      bool do_relu = kReluAll || p.relu != 0;
      float ymul = 1.f;
      if (cur.valid && (p.relu_inactive_coarse || p.ymask_coarse)) {
        const RowPos& rp = cur.rp;
        const int cell = (rp.n * p.cells_h + rp.y / p.patch_h) * p.cells_w + rp.x / p.patch_w;
        if (!kReluAll && p.relu_inactive_coarse) do_relu = p.relu_inactive_coarse[cell] == 0;
        if (p.ymask_coarse) ymul = p.ymask_coarse[cell] ? 1.f : 0.f;
      }
      // next tile's rows and vectors: issue the global loads now, use them later
      int tn = next_valid(t + t_step);  // this group's next tile: EG tiles on
      for (int g = 1; g < L::EG && tn < tiles; ++g) tn = next_valid(tn + t_step);
      RowInfo nxt = cur;
      VecPre vpn;
      int raw_n = 0;
      if (tn < tiles) {
        raw_n = row_raw(tn);
        if (!cached) vpn = vec_load(tn);
      }
      const float* const vbi = cached ? bias_cache + c_base : vbi_w;
      float pd = 0.f;  // this row's partial dot with the next masker
      mbar_wait(&acc_full[acc], acc_phase);
      if (trc && ew == 0 && lane == 0 && local < 1024) trc[TRACE_EPI + 4 * local] = global_ns();
      tc_fence_after();
      if (pre) asm volatile("cp.async.wait_group 0;" ::: "memory");
      if (tma_out) bulk_wait_read<0>();  // staging rows of an earlier TMA store are free
      __syncwarp();
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + col0;
      if (KS > 1) {
        // split-K: this CTA's fp32 partial of its rows -> its own operand smem
        // (every MMA of the tile has completed); reduced after the role loops
        float* prow = reinterpret_cast<float*>(base + L::A_OFF) + (size_t)(q * 32 + lane) * (BN + 4) + col0;
#pragma unroll 1
        for (int j = 0; j < EW_COLS / CH; ++j) {
          uint32_t r[CH];
          tmem_ld_32x32b<CH>(tbase + j * CH, r);
#pragma unroll
          for (int e = 0; e < CH; e += 4)
            *reinterpret_cast<float4*>(prow + j * CH + e) = make_float4(
                __uint_as_float(r[e]), __uint_as_float(r[e + 1]), __uint_as_float(r[e + 2]), __uint_as_float(r[e + 3]));
        }
        break;  // one tile per cluster
      }
      auto slot_of = [&](int cl) { return reinterpret_cast<uint4*>(stg + soff(lane, cl >> 3)); };
      // generic 8-column step: affine, masks, residual, ReLU, store
      auto finish8 = [&](const uint32_t* rv, int cl) {
        float v[8];
        const float4 b0 = *reinterpret_cast<const float4*>(vbi + cl);
        const float4 b1 = *reinterpret_cast<const float4*>(vbi + cl + 4);
        float4 s0 = make_float4(1.f, 1.f, 1.f, 1.f), s1 = s0;
        if (has_scale) {
          s0 = *reinterpret_cast<const float4*>(vsc + cl);
          s1 = *reinterpret_cast<const float4*>(vsc + cl + 4);
        }
        v[0] = fmaf(__uint_as_float(rv[0]), s0.x, b0.x);
        v[1] = fmaf(__uint_as_float(rv[1]), s0.y, b0.y);
        v[2] = fmaf(__uint_as_float(rv[2]), s0.z, b0.z);
        v[3] = fmaf(__uint_as_float(rv[3]), s0.w, b0.w);
        v[4] = fmaf(__uint_as_float(rv[4]), s1.x, b1.x);
        v[5] = fmaf(__uint_as_float(rv[5]), s1.y, b1.y);
        v[6] = fmaf(__uint_as_float(rv[6]), s1.z, b1.z);
        v[7] = fmaf(__uint_as_float(rv[7]), s1.w, b1.w);
        if (p.ymask_channel) {
          const uint2 mk = __ldg(reinterpret_cast<const uint2*>(
              p.ymask_channel + (size_t)cur.rp.n * p.n_out + c_base + cl));
#pragma unroll
          for (int e = 0; e < 8; ++e)
            v[e] *= ((e < 4 ? (mk.x >> (8 * e)) : (mk.y >> (8 * (e - 4)))) & 0xff) ? 1.f : 0.f;
        }
        if (p.ymask_coarse) {
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] *= ymul;
        }
        uint4* slot = slot_of(cl);
        if (pre) {
          const uint4 rr = *slot;
          float2 f;
          f = unpack_bf16x2(rr.x); v[0] += f.x; v[1] += f.y;
          f = unpack_bf16x2(rr.y); v[2] += f.x; v[3] += f.y;
          f = unpack_bf16x2(rr.z); v[4] += f.x; v[5] += f.y;
          f = unpack_bf16x2(rr.w); v[6] += f.x; v[7] += f.y;
        }
        if (do_relu) {
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = fmaxf(v[e], 0.f);
        }
        if (!staged) {
          float* o = reinterpret_cast<float*>(p.out) + cur.dst * p.out_ld + c_base + cl;
          reinterpret_cast<float4*>(o)[0] = make_float4(v[0], v[1], v[2], v[3]);
          reinterpret_cast<float4*>(o)[1] = make_float4(v[4], v[5], v[6], v[7]);
        } else {
          uint4 w;
          w.x = pack_bf16x2(v[0], v[1]);
          w.y = pack_bf16x2(v[2], v[3]);
          w.z = pack_bf16x2(v[4], v[5]);
          w.w = pack_bf16x2(v[6], v[7]);
          *slot = w;
          if (!kPlain && p.mdot_w) {  // the stored (bf16) values are what the next masker sees
            const float4 n0 = *reinterpret_cast<const float4*>(vnw + cl);
            const float4 n1 = *reinterpret_cast<const float4*>(vnw + cl + 4);
            float2 f;
            f = unpack_bf16x2(w.x); pd = fmaf(f.x, n0.x, pd); pd = fmaf(f.y, n0.y, pd);
            f = unpack_bf16x2(w.y); pd = fmaf(f.x, n0.z, pd); pd = fmaf(f.y, n0.w, pd);
            f = unpack_bf16x2(w.z); pd = fmaf(f.x, n1.x, pd); pd = fmaf(f.y, n1.y, pd);
            f = unpack_bf16x2(w.w); pd = fmaf(f.x, n1.z, pd); pd = fmaf(f.y, n1.w, pd);
          }
        }
      };
      // branch-free CH-column step of the plain epilogue: y = acc + bias (+ resid), ReLU
      auto plain_chunk = [&](const uint32_t* rv, int cl, bool with_resid, bool relu) {
        uint4 rr[CH / 8];
        if (with_resid) {
#pragma unroll
          for (int g = 0; g < CH / 8; ++g) rr[g] = *slot_of(cl + g * 8);
        }
#pragma unroll
        for (int g = 0; g < CH / 8; ++g) {
          const float4 b0 = *reinterpret_cast<const float4*>(vbi + cl + g * 8);
          const float4 b1 = *reinterpret_cast<const float4*>(vbi + cl + g * 8 + 4);
          float v[8];
          v[0] = __uint_as_float(rv[g * 8 + 0]) + b0.x;
          v[1] = __uint_as_float(rv[g * 8 + 1]) + b0.y;
          v[2] = __uint_as_float(rv[g * 8 + 2]) + b0.z;
          v[3] = __uint_as_float(rv[g * 8 + 3]) + b0.w;
          v[4] = __uint_as_float(rv[g * 8 + 4]) + b1.x;
          v[5] = __uint_as_float(rv[g * 8 + 5]) + b1.y;
          v[6] = __uint_as_float(rv[g * 8 + 6]) + b1.z;
          v[7] = __uint_as_float(rv[g * 8 + 7]) + b1.w;
          if (p.ymask_channel) {  // per-sample channel mask (dense-masked channel schedule)
            const uint2 mk = __ldg(reinterpret_cast<const uint2*>(
                p.ymask_channel + (size_t)cur.rp.n * p.n_out + c_base + cl + g * 8));
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (!(((e < 4 ? (mk.x >> (8 * e)) : (mk.y >> (8 * (e - 4)))) & 0xff))) v[e] = 0.f;
          }
          if (with_resid) {
            float2 f;
            f = unpack_bf16x2(rr[g].x); v[0] += f.x; v[1] += f.y;
            f = unpack_bf16x2(rr[g].y); v[2] += f.x; v[3] += f.y;
            f = unpack_bf16x2(rr[g].z); v[4] += f.x; v[5] += f.y;
            f = unpack_bf16x2(rr[g].w); v[6] += f.x; v[7] += f.y;
          }
          if (relu) {
#pragma unroll
            for (int e = 0; e < 8; ++e) v[e] = fmaxf(v[e], 0.f);
          }
          uint4 w;
          w.x = pack_bf16x2(v[0], v[1]);
          w.y = pack_bf16x2(v[2], v[3]);
          w.z = pack_bf16x2(v[4], v[5]);
          w.w = pack_bf16x2(v[6], v[7]);
          *slot_of(cl + g * 8) = w;
        }
      };
      const bool full = nch == EW_COLS;
#pragma unroll 1
      for (int j = 0; j < EW_COLS / CH; ++j) {
        if (j * CH >= nch) break;
        uint32_t r[CH];
        if (ti.kb_hi > ti.kb_lo && !(p.dbg & 4)) {
          tmem_ld_32x32b<CH>(tbase + j * CH, r);
        } else {  // empty K (no channel kept): y = 0
#pragma unroll
          for (int e = 0; e < CH; ++e) r[e] = 0u;
        }
        if (!cur.valid || (p.dbg & 1)) continue;
        if (kPlain || (plain && full)) {
          if (pre) {
            if (do_relu) plain_chunk(r, j * CH, true, true);
            else plain_chunk(r, j * CH, true, false);
          } else {
            if (do_relu) plain_chunk(r, j * CH, false, true);
            else plain_chunk(r, j * CH, false, false);
          }
        } else if constexpr (!kPlain) {
#pragma unroll
          for (int g = 0; g < CH / 8; ++g) {
            if (j * CH + g * 8 >= nch) break;
            finish8(r + g * 8, j * CH + g * 8);
          }
        }
      }
      if (!kPlain && p.mdot_w) {
        // rows of one patch are consecutive lanes: reduce per patch, one atomic each
        const int seg = p.patch_h * p.patch_w;
        if (seg <= 32 && (32 % seg) == 0) {
          for (int o = 1; o < seg; o <<= 1) pd += __shfl_xor_sync(0xffffffffu, pd, o);
          if (cur.valid && (lane % seg) == 0) {
            const RowPos& rp = cur.rp;
            atomicAdd(p.mdot_out + (rp.n * p.cells_h + rp.y / p.patch_h) * p.cells_w +
                          rp.x / p.patch_w, pd);
          }
        } else if (cur.valid) {
          const RowPos& rp = cur.rp;
          atomicAdd(p.mdot_out + (rp.n * p.cells_h + rp.y / p.patch_h) * p.cells_w +
                        rp.x / p.patch_w, pd);
        }
      }
      // accumulator consumed: hand the TMEM buffer back to the MMA warp early
      if (trc && ew == 0 && lane == 0 && local < 1024) trc[TRACE_EPI + 4 * local + 1] = global_ns();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {  // one arrive per warp, on the leader's barrier
        if constexpr (PAIR)
          mbar_arrive_cluster(mapa_shared(smem_u32(&acc_empty[acc]), 0));
        else
          mbar_arrive(&acc_empty[acc]);
      }
      __syncwarp();
      if (tn < tiles) {
        nxt = row_info(tn, raw_n);
        if (!cached) vec_store(vpn);  // this tile's vector reads are done (syncwarp above)
        // with two staging buffers the next residual streams in now
        if (pre && kDoubleStage) prefetch(tn, nxt, (local + 1) & 1);
      }
      if (tma_out && vchunks > 0 && !(p.dbg & 2)) {
        // the warp's 32 staged rows leave as TMA boxes: one 32-row box (dense
        // rows) or one S x S pixel box per active patch (scattered patches)
        fence_proxy_async_smem();
        __syncwarp();
        const uint32_t sl = base_u32 + stg_off0 + buf * L::STG_BUF;
        if (p.tma_out == 1) {
          if (lane == 0) tma_store_2d(&tmap_o, sl, c_base, (t / n_tiles) * MT + rank * BM + q * 32);
        } else if (cur.valid && lane % (p.patch_h * p.patch_w) == 0) {
          int y = cur.rp.y;
          if (p.misplace_first && cur.fp) y = (y + p.patch_h) % p.out_h;
          tma_store_4d(&tmap_o, sl + lane * SROW, c_base, cur.rp.x, y, cur.rp.n);
        }
        bulk_commit();
      } else if (staged && vchunks > 0 && !(p.dbg & 2)) {
        // row-major sweep of the staged 32 x EW_COLS slice: each instruction
        // writes 32 / CPR whole row segments
        constexpr int RPI = 32 / CPR;  // rows per warp instruction
        const int cc = lane % CPR;
        const int rr0 = lane / CPR;
#pragma unroll 8
        for (int it2 = 0; it2 < CPR; ++it2) {
          const int r = it2 * RPI + rr0;
          const int rv = __shfl_sync(0xffffffffu, (int)cur.valid, r);
          const long long dr = __shfl_sync(0xffffffffu, cur.dst, r);
          if (rv && cc < vchunks)
            *reinterpret_cast<uint4*>(outp + dr * p.out_ld + c_base + cc * 8) =
                *reinterpret_cast<const uint4*>(stg + soff(r, cc));
        }
      }
      __syncwarp();
      if (trc && ew == 0 && lane == 0 && local < 1024) trc[TRACE_EPI + 4 * local + 2] = global_ns();
      if (tn < tiles && pre && !kDoubleStage) prefetch(tn, nxt, 0);
      cur = nxt;
      t = tn;
    }
    if (tma_out) bulk_wait_all();  // stores done before the CTA's shared memory goes away
  }

  if (KS > 1) {
    // split-K reduction through distributed shared memory: CTA ks finishes rows
    // [ks*BM/KS, (ks+1)*BM/KS) of the cluster's tile, adding the KS partials in
    // rank order (deterministic), then bias [+ residual] [+ ReLU] and the store
    cluster_sync();
    const int t = t_begin;
    if (warp >= FIRST_EPI && t < tiles) {
      const TileInfo ti = tile_info<BN, PAIR>(p, t, n_tiles, rank);
      const int ks = (int)cluster_ctarank();
      const int rows = BM / KS, r0 = ks * rows;
      const float* bias_cache = reinterpret_cast<const float*>(base + L::VEC_OFF);
      const __nv_bfloat16* resid = reinterpret_cast<const __nv_bfloat16*>(p.resid);
      __nv_bfloat16* outp = reinterpret_cast<__nv_bfloat16*>(p.out);
      constexpr bool kRes = EP == EP_PLAIN_RES || EP == EP_PLAIN_RES_RELU;
      const bool relu = EP == EP_PLAIN_RELU || EP == EP_PLAIN_RES_RELU || p.relu != 0;
      const uint32_t part0 = base_u32 + L::A_OFF;
      for (int item = threadIdx.x - FIRST_EPI * 32; item < rows * (BN / 8); item += NUM_EPI_WARPS * 32) {
        const int r = r0 + item / (BN / 8), c8 = item % (BN / 8);
        const int col = ti.n0 + c8 * 8;
        if (col >= p.n_out) continue;
        const int m = ti.m0 + r;
        RowPos rp;
        bool fp;
        if (!map_row_raw(p, m, nvalid, row_fetch(p, m), rp, fp)) continue;
        long long dst = m;
        if (p.out_mode != OUT_ROW) {
          int y = rp.y;
          if (p.misplace_first && fp) y = (y + p.patch_h) % p.out_h;
          dst = (long long)(rp.n * p.out_h + y) * p.out_w + rp.x;
        }
        float v[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const uint32_t off = (uint32_t)((r * (BN + 4) + c8 * 8) * 4);
        for (int k = 0; k < KS; ++k) {
          float4 a, b;
          const uint32_t ad = mapa_shared(part0 + off, (uint32_t)k);
          asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w) : "r"(ad));
          asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w) : "r"(ad + 16u));
          v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w;
          v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] += bias_cache[col + e];
        if (kRes) {
          const uint4 rr = *reinterpret_cast<const uint4*>(resid + dst * p.resid_ld + col);
          float2 f;
          f = unpack_bf16x2(rr.x); v[0] += f.x; v[1] += f.y;
          f = unpack_bf16x2(rr.y); v[2] += f.x; v[3] += f.y;
          f = unpack_bf16x2(rr.z); v[4] += f.x; v[5] += f.y;
          f = unpack_bf16x2(rr.w); v[6] += f.x; v[7] += f.y;
        }
        if (relu) {
#pragma unroll
          for (int e = 0; e < 8; ++e) v[e] = fmaxf(v[e], 0.f);
        }
        uint4 w;
        w.x = pack_bf16x2(v[0], v[1]);
        w.y = pack_bf16x2(v[2], v[3]);
        w.z = pack_bf16x2(v[4], v[5]);
        w.w = pack_bf16x2(v[6], v[7]);
        *reinterpret_cast<uint4*>(outp + dst * p.out_ld + col) = w;
      }
    }
    cluster_sync();  // peers done reading this CTA's partials
  }

  tc_fence_before();
  if constexpr (PAIR)
    cluster_sync();  // the peer's smem / barriers must outlive the leader's last use
  else
    __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    if constexpr (PAIR)
      tmem_dealloc_pair<L::TMEM_COLS>(tmem_base);
    else
      tmem_dealloc<L::TMEM_COLS>(tmem_base);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

template <int BN, int STAGES, int NSTG, bool PAIR = false, int AM = AM_ANY, int EP = EP_ANY>
static cudaError_t launch_bn(const CUtensorMap& tmap_a, const CUtensorMap& tmap, const CUtensorMap& tmap_o,
                             const ConvParams& p, int tiles_max,
                             int num_sms, cudaStream_t stream) {
  using L = Smem<BN, STAGES, NSTG, PAIR>;
  static_assert(L::ALLOC <= 227 * 1024, "shared memory budget");
  auto kern = conv_gemm_kernel<BN, STAGES, NSTG, PAIR, AM, EP>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::ALLOC);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  static const int grid_env = [] {
    const char* e = getenv("LAUD_GRID");  // debug: cap the persistent grid
    return e ? atoi(e) : 0;
  }();
  // persistent grid: one CTA (PAIR: one CTA pair per TPC) per SM
  const int units = PAIR ? num_sms / 2 : num_sms;
  int grid = tiles_max < units ? tiles_max : units;
  if (grid_env > 0 && grid > grid_env) grid = grid_env;
  if (grid < 1) grid = 1;
  if (!PAIR && p.ksplit > 1) {  // cluster split-K: one tile per cluster of ksplit CTAs
    if (BN != 64 || EP == EP_ANY || BM * (BN + 4) * 4 > L::STG_OFF || tiles_max * p.ksplit > num_sms)
      return cudaErrorInvalidValue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(tiles_max * p.ksplit, 1, 1);
    cfg.blockDim = dim3(NUM_THREADS, 1, 1);
    cfg.dynamicSmemBytes = L::ALLOC;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.ksplit;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, tmap_a, tmap, tmap_o, p);
  }
  if constexpr (PAIR) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * grid, 1, 1);
    cfg.blockDim = dim3(NUM_THREADS, 1, 1);
    cfg.dynamicSmemBytes = L::ALLOC;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, tmap_a, tmap, tmap_o, p);
  } else {
    return launch_k(kern, dim3(grid), dim3(NUM_THREADS), L::ALLOC, stream, tmap_a, tmap, tmap_o, p);
  }
}

// One translation unit per tile width instantiates that width's kernels
// (conv_gemm_bn*.cu, compiled in parallel); conv_gemm.cu dispatches.
struct ConvLaunch {
  const CUtensorMap* tmap_a;
  const CUtensorMap* tmap_b;
  const CUtensorMap* tmap_o;  // output rows for the TMA-store epilogue (ConvParams::tma_out)
  const ConvParams* p;
  int tiles_max, num_sms, am;
  bool ep_plain, relu_all;
  cudaStream_t stream;
};

#define LAUD_LB(B, S, N, A)                                                                                     \
  (!c.ep_plain ? launch_bn<B, S, N, false, A, EP_ANY>(*c.tmap_a, *c.tmap_b, *c.tmap_o, *c.p, c.tiles_max, c.num_sms, c.stream) \
   : c.p->resid                                                                                                 \
       ? (c.relu_all ? launch_bn<B, S, N, false, A, EP_PLAIN_RES_RELU>(*c.tmap_a, *c.tmap_b, *c.tmap_o, *c.p, c.tiles_max, c.num_sms, c.stream) \
                     : launch_bn<B, S, N, false, A, EP_PLAIN_RES>(*c.tmap_a, *c.tmap_b, *c.tmap_o, *c.p, c.tiles_max, c.num_sms, c.stream))   \
       : (c.relu_all ? launch_bn<B, S, N, false, A, EP_PLAIN_RELU>(*c.tmap_a, *c.tmap_b, *c.tmap_o, *c.p, c.tiles_max, c.num_sms, c.stream)     \
                     : launch_bn<B, S, N, false, A, EP_PLAIN>(*c.tmap_a, *c.tmap_b, *c.tmap_o, *c.p, c.tiles_max, c.num_sms, c.stream)))
#define LAUD_BN_DISPATCH(B, S, N)                             \
  switch (c.am) {                                             \
    case AM_TILE: return LAUD_LB(B, S, N, AM_TILE);           \
    case AM_TILE_DOT: return LAUD_LB(B, S, N, AM_TILE_DOT);   \
    case AM_BOX: return LAUD_LB(B, S, N, AM_BOX);             \
    case AM_G4: return LAUD_LB(B, S, N, AM_G4);               \
    default: return LAUD_LB(B, S, N, AM_ANY);                 \
  }

cudaError_t launch_conv_bn64(const ConvLaunch& c);
cudaError_t launch_conv_bn128(const ConvLaunch& c);
cudaError_t launch_conv_bn256(const ConvLaunch& c);
cudaError_t launch_conv_pair(const ConvLaunch& c, int pair);

}  // namespace laud
