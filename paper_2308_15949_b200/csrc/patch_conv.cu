// Patch conv2 with the halo in shared memory (sm_100a): the 3x3 convolution
// over the active S x S patches of LAUDNet's gather-conv-scatter schedule
// (`reference.py:384-398`: per active cell, gather the (S-1)*stride+3 halo
// window of conv1's output, convolve "valid", keep the S x S result).
//
// The reference re-reads overlapping halos per tap ("input patches overlap,
// leading to repeated loads").  Here each patch's halo is
// loaded into shared memory ONCE per 64-channel block and all nine taps read
// it in place: the halo of P = 128/S patches is stored position-major,
//     halo row (y, x, p) at ((y * E + x) * P + p) * 128 bytes  (E = S + 2),
// so for a tap (ky, kx) and patch row ly the 128 GEMM rows (lx, p), lx < S,
// p < P, are halo rows ((ly + ky) * E + kx + lx) * P + p — one contiguous,
// uniformly strided run of 128 rows.  The tcgen05 A operand is therefore a
// plain SW128 K-major descriptor pointing into the halo: no im2col copies,
// no per-tap gathers.  A tile is P patches x S^2 pixels: S accumulators
// (one per patch row ly) of 128 x BN fp32 in TMEM share every B stage, so
// each weight tile streamed from L2 feeds 128*S output rows.
//
// Halo fill: TMA tile::gather4 (4 patches' pixels of one halo position per
// op; out-of-image pixels are out-of-bounds rows -> zero fill, i.e. conv2's
// zero padding).  The halo is split into E bands (one halo input row y of
// every patch); band y is released as soon as the last tap reading it
// (ky = min(y, 2)) has been issued, so the next channel block's bands
// stream in underneath the current block's remaining taps.
//
// Warp roles (512 threads): warps 0-3 halo producers, warp 4 B (weights)
// TMA, warp 5 MMA issuer, warps 6-15 ... epilogue (tcgen05.ld -> scale/bias
// /ReLU -> bf16 -> smem staging -> coalesced row stores to the compact h2
// rows, patch-major order (m = patch * S^2 + ly * S + lx) exactly as the
// generic engine writes them, so conv3 + scatter-add is unchanged).
#include <cuda.h>
#include <cuda_runtime.h>

#include "laud_conv.cuh"
#include "laud_launch.cuh"
#include "laud_ptx.cuh"
#include "laud_rows.cuh"

namespace laud {
namespace pc {

#ifndef LAUD_PC_PROD
#define LAUD_PC_PROD 4
#endif
constexpr int NUM_PROD = LAUD_PC_PROD;  // halo producer warps (TMA issue is serial per warp)
constexpr int NUM_EPI = 8;              // epilogue warps
constexpr int WARP_B = NUM_PROD, WARP_MMA = NUM_PROD + 1;
constexpr int FIRST_EPI = NUM_PROD + 2;
constexpr int THREADS = (FIRST_EPI + NUM_EPI) * 32;

template <int S, int BN>
struct Cfg {
  static constexpr int P = 128 / S;            // patches per tile
  static constexpr int E = S + 2;              // halo edge (3x3, stride 1)
  static constexpr int BAND_ROWS = E * P;      // one halo input row of every patch
  static constexpr int BAND_BYTES = BAND_ROWS * 128;
  static constexpr int HALO_BYTES = E * BAND_BYTES;
  static constexpr int TILE_COLS = S * BN;     // TMEM columns of one tile's accumulators
  static constexpr int NBUF = 2 * TILE_COLS <= 512 ? 2 : 1;
  static constexpr uint32_t TMEM_COLS = NBUF * TILE_COLS <= 32 ? 32 : NBUF * TILE_COLS <= 64 ? 64
                                        : NBUF * TILE_COLS <= 128 ? 128 : NBUF * TILE_COLS <= 256 ? 256 : 512;
  static constexpr int B_STAGE = BN * 64 * 2;
  static constexpr int EW_COLS = BN / (NUM_EPI / 4);  // columns per epilogue warp
  static constexpr int STG_ROW = EW_COLS * 2 + 16;    // padded staging row slice (bytes)
  static constexpr int STG_WARP = 32 * STG_ROW;
  static constexpr int STG_BYTES = NUM_EPI * STG_WARP;
  static constexpr int VEC_FLOATS = 2 * 512;          // scale, bias (n_out <= 512)
  static constexpr int FIXED = HALO_BYTES + STG_BYTES + VEC_FLOATS * 4 + 1024 + 256;
  static constexpr int STAGES_FIT = (227 * 1024 - FIXED) / B_STAGE;
  static constexpr int STAGES = STAGES_FIT > 6 ? 6 : STAGES_FIT;
  static constexpr int HALO_OFF = 0;
  static constexpr int B_OFF = HALO_OFF + HALO_BYTES;
  static constexpr int STG_OFF = B_OFF + STAGES * B_STAGE;
  static constexpr int VEC_OFF = STG_OFF + STG_BYTES;
  static constexpr int BAR_OFF = VEC_OFF + VEC_FLOATS * 4;
  static constexpr int NUM_BARS = 2 * E + 2 * STAGES + 2 * NBUF;
  static constexpr int TMEM_SLOT_OFF = BAR_OFF + NUM_BARS * 8;
  static constexpr int ALLOC = TMEM_SLOT_OFF + 16 + 1024;
  static_assert(STAGES >= 2, "shared memory: fewer than two weight stages");
  // split-K partials [S*128 rows][PSTRIDE fp32] reuse the halo + weight stages
  static constexpr int PSTRIDE = BN + 4;  // +16 B: conflict-free row-per-lane float4 stores
  static constexpr bool SPLIT_OK = S * 128 * PSTRIDE * 4 <= STG_OFF;  // else split-K is not offered
  static_assert(ALLOC <= 227 * 1024, "shared memory budget");
  static_assert(EW_COLS % 16 == 0, "epilogue slice");
};

template <int S, int BN>
__global__ void __launch_bounds__(THREADS, 1)
    patch_conv_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                      const ConvParams p) {
  using L = Cfg<S, BN>;
  constexpr int P = L::P, E = L::E;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  const uint32_t base_u32 = (raw_u32 + 1023u) & ~1023u;
  uint8_t* base = smem_raw + (base_u32 - raw_u32);
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + L::BAR_OFF);
  uint64_t* band_full = bars;
  uint64_t* band_empty = bars + E;
  uint64_t* full = bars + 2 * E;
  uint64_t* empty = full + L::STAGES;
  uint64_t* acc_full = empty + L::STAGES;
  uint64_t* acc_empty = acc_full + L::NBUF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(base + L::TMEM_SLOT_OFF);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int OPS = E * (P / 4);  // gather4 ops per band
  static_assert(OPS <= 32 * NUM_PROD, "one gather4 per producer thread per band");

  if (threadIdx.x == 0) {
    for (int y = 0; y < E; ++y) {
      mbar_init(&band_full[y], 1);
      mbar_init(&band_empty[y], 1);
    }
    for (int s = 0; s < L::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < L::NBUF; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], NUM_EPI);
    }
    fence_barrier_init();
  }
  if (warp == WARP_B && lane == 0) {
    tma_prefetch_desc(&tmap_a);
    tma_prefetch_desc(&tmap_b);
  }
  if (warp == WARP_MMA) tmem_alloc<L::TMEM_COLS>(tmem_slot);
  // per-column scale / bias for the whole kernel (n_out <= 512, host-checked)
  float* vsc = reinterpret_cast<float*>(base + L::VEC_OFF);
  float* vbi = vsc + 512;
  pdl_wait();  // conv1's output and the cell list are read from here on
  if (warp >= FIRST_EPI) {
    for (int i = threadIdx.x - FIRST_EPI * 32; i < p.n_out; i += NUM_EPI * 32) {
      vsc[i] = p.scale ? __ldg(p.scale + i) : 1.f;
      vbi[i] = p.bias ? __ldg(p.bias + i) : 0.f;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  pdl_trigger();
  const uint32_t tmem_base = *tmem_slot;

  const int s2 = S * S;
  const int count = p.count ? min(__ldg(p.count) * max(p.list_expand, 1), p.rows_max / s2)
                            : p.rows_max / s2;  // active patches
  const int n_tiles = (p.n_out + BN - 1) / BN;
  const int m_tiles = (count + P - 1) / P;
  const int tiles = m_tiles * n_tiles;
  const int ncb = p.kpad / 64;  // channel blocks
  // Work schedule.  Items are (tile, part): a part item is a split-K slice of a
  // tile shared by the CTAs of a cluster (fp32 partials reduced through DSMEM
  // after the role loops).
  //  * small grids (ksplit = KS > 1): every tile split KS ways, one wave;
  //  * tail split (clusters of 2): whole tiles round-robin over the CTAs for
  //    the complete waves, then the last partial wave's tiles (at most one per
  //    cluster) split over the cluster's 2 CTAs — the tail costs half a tile
  //    instead of a whole one (e.g. 196 tiles on 148 SMs: 1.5 instead of 2);
  //  * otherwise whole tiles round-robin.
  const int KS = (L::SPLIT_OK && p.ksplit > 1) ? p.ksplit : 1;
  const bool tail = L::SPLIT_OK && KS == 1 && p.tail_split;
  const int ks = (KS > 1 || tail) ? (int)cluster_ctarank() : 0;
  const int NP = KS > 1 ? KS : 2;  // parts of a split tile
  const int t_begin = blockIdx.x / KS, t_step = gridDim.x / KS;
  int F = tiles, split_t = -1;
  if (tail) {
    const int n_cta = gridDim.x, rounds = tiles / n_cta, R = tiles - rounds * n_cta;
    if (R > 0 && R <= n_cta / 2) {
      F = rounds * n_cta;
      split_t = (int)blockIdx.x / 2 < R ? F + (int)blockIdx.x / 2 : -1;
    }
  }
  const int nfull = F > (int)blockIdx.x ? (F - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  auto work = [&](int k, int& t, bool& part) -> bool {
    if (KS > 1) {
      t = t_begin + k * t_step;
      part = true;
      return t < tiles;
    }
    if (k < nfull) {
      t = blockIdx.x + k * gridDim.x;
      part = false;
      return true;
    }
    t = split_t;
    part = true;
    return k == nfull && split_t >= 0;
  };
  // channel blocks of item (t, part) for this CTA: all of them, or (grouped
  // conv) only those holding the input channels of the groups the tile's N
  // range spans (the block-diagonal weights are zero elsewhere); a part item
  // takes this CTA's slice
  auto cb_range = [&](int t, bool part, int& b0, int& b1) {
    int lo = 0, hi = ncb;
    if (p.groups > 1) {
      const int n0 = (t % n_tiles) * BN;
      const int g0 = n0 / p.gw_out;
      const int g1 = min(p.groups, (min(n0 + BN, p.n_out) + p.gw_out - 1) / p.gw_out);
      lo = (g0 * p.gw_in) / 64;
      hi = (g1 * p.gw_in + 63) / 64;
    }
    if (!part) {
      b0 = lo;
      b1 = hi;
      return;
    }
    b0 = lo + ks * (hi - lo) / NP;
    b1 = lo + (ks + 1) * (hi - lo) / NP;
  };

  if (warp < NUM_PROD) {
    // ---------------------------------------------------------------- halo producers
    const int tid = threadIdx.x;
    // op j = lane * NUM_PROD + warp: the band's gather4 issues are spread evenly
    // over the producer warps (each warp issues its lanes' TMA ops serially)
    const int op = lane * NUM_PROD + warp;
    const bool issuer = op < OPS;
    const int xpos = op / (P / 4);  // halo column of this thread's op
    const int quad = op % (P / 4);  // 4 patches p = 4*quad .. 4*quad+3
    const int cpi = p.cells_h * p.cells_w;
    uint32_t fill = 0;  // band fills so far (same sequence for every band)
    int t;
    bool part;
    for (int k = 0; work(k, t, part); ++k) {
      const int mt = t / n_tiles;
      int pn[4], py[4], px[4];
      bool pv[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int pi = mt * P + quad * 4 + j;
        pv[j] = issuer && pi < count;
        pn[j] = 0, py[j] = 0, px[j] = 0;
        if (pv[j]) {
          const int cell = list_cell(p, pi);
          pn[j] = cell / cpi;
          const int cr = cell - pn[j] * cpi;
          const int ci = cr / p.cells_w;
          py[j] = ci * S - 1;                       // halo origin on conv1's grid (pad 1)
          px[j] = (cr - ci * p.cells_w) * S - 1 + xpos;
        }
      }
      int cb0, cb1;
      cb_range(t, part, cb0, cb1);
      for (int cb = cb0; cb < cb1; ++cb, ++fill) {
        for (int y = 0; y < E; ++y) {
          mbar_wait(&band_empty[y], (fill & 1) ^ 1);
          const uint32_t dst = base_u32 + L::HALO_OFF + y * L::BAND_BYTES + (xpos * P + quad * 4) * 128;
          if (tid == 0) mbar_arrive_expect_tx(&band_full[y], L::BAND_BYTES);
          if (issuer) {
            int r[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int iy = py[j] + y, ix = px[j];
              r[j] = (pv[j] && iy >= 0 && iy < p.in_h && ix >= 0 && ix < p.in_w)
                         ? (pn[j] * p.in_h + iy) * p.in_w + ix
                         : p.a_rows;  // out of bounds -> zeros (padding / no patch)
            }
            tma_gather4(dst, &tmap_a, &band_full[y], cb * 64, r[0], r[1], r[2], r[3]);
          }
        }
      }
    }
  } else if (warp == WARP_B) {
    // ---------------------------------------------------------------- weights (B) TMA
    if (lane == 0) {
      uint32_t it = 0;
      int t;
      bool part;
      for (int k = 0; work(k, t, part); ++k) {
        const int n0 = (t % n_tiles) * BN;
        int cb0, cb1;
        cb_range(t, part, cb0, cb1);
        for (int cb = cb0; cb < cb1; ++cb)
          for (int tap = 0; tap < 9; ++tap, ++it) {
            const int stage = it % L::STAGES;
            mbar_wait(&empty[stage], ((it / L::STAGES) & 1) ^ 1);
            mbar_arrive_expect_tx(&full[stage], L::B_STAGE);
            tma_load_2d(base_u32 + L::B_OFF + stage * L::B_STAGE, &tmap_b, &full[stage], tap * p.kpad + cb * 64, n0);
          }
      }
    }
  } else if (warp == WARP_MMA) {
    // ---------------------------------------------------------------- MMA issuer
    constexpr uint32_t idesc = umma_idesc_bf16(128, BN);
    uint32_t it = 0, fill = 0, local = 0;
    int t;
    bool part;
    for (int k = 0; work(k, t, part); ++k, ++local) {
      const int buf = local % L::NBUF;
      mbar_wait(&acc_empty[buf], ((local / L::NBUF) & 1) ^ 1);
      tc_fence_after();
      const uint32_t tacc = tmem_base + buf * L::TILE_COLS;
      int cb0, cb1;
      cb_range(t, part, cb0, cb1);
      for (int cb = cb0; cb < cb1; ++cb, ++fill) {
        for (int ky = 0; ky < 3; ++ky) {
          // bands first read at this ky: 0 .. S-1 at ky = 0, then ky + S - 1
          for (int y = (ky == 0 ? 0 : ky + S - 1); y <= ky + S - 1; ++y) mbar_wait(&band_full[y], fill & 1);
          for (int kx = 0; kx < 3; ++kx, ++it) {
            const int stage = it % L::STAGES;
            mbar_wait(&full[stage], (it / L::STAGES) & 1);
            tc_fence_after();
            if (lane == 0) {
              const uint32_t sb = base_u32 + L::B_OFF + stage * L::B_STAGE;
#pragma unroll
              for (int ly = 0; ly < S; ++ly) {
                const uint32_t sa = base_u32 + L::HALO_OFF + (ky + ly) * L::BAND_BYTES + kx * P * 128;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  umma_bf16(tacc + ly * BN, umma_sdesc_sw128(sa + k * 32), umma_sdesc_sw128(sb + k * 32), idesc,
                            cb != cb0 || (ky | kx | k) != 0);
              }
              umma_commit(&empty[stage]);
              // bands whose last reader was this ky go back to the producers
              if (kx == 2) {
                if (ky < 2) {
                  umma_commit(&band_empty[ky]);
                } else {
                  for (int y = 2; y < E; ++y) umma_commit(&band_empty[y]);
                }
              }
            }
            __syncwarp();
          }
        }
      }
      if (lane == 0) umma_commit(&acc_full[buf]);
      __syncwarp();
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    // warp e: TMEM lane quadrant q = warp % 4 (hardware restriction), columns
    // [cs * EW_COLS, +EW_COLS) of each of the tile's S accumulators.  Lane i
    // of quadrant q holds GEMM row (lx, p) = divmod(32q + i, P).
    constexpr int EW = L::EW_COLS;
    constexpr int CPR = EW / 8;       // 16-byte chunks per row slice
    constexpr int CH = EW < 32 ? EW : 32;
    const int ew = warp - FIRST_EPI;
    const int q = warp & 3;
    const int cs = ew >> 2;
    const int col0 = cs * EW;
    uint8_t* stg = base + L::STG_OFF + ew * L::STG_WARP;
    __nv_bfloat16* outp = reinterpret_cast<__nv_bfloat16*>(p.out);
    const int i = q * 32 + lane;
    const int lx = i / P, pl = i - (i / P) * P;
    uint32_t local = 0;
    int t;
    bool part;
    for (int k = 0; work(k, t, part); ++k, ++local) {
      const int buf = local % L::NBUF;
      const int mt = t / n_tiles;
      if (part) {
        // split-K: this CTA's fp32 partial -> its own smem (the halo / weight
        // region: every MMA of the tile has completed), reduced after the
        // cluster barrier below
        mbar_wait(&acc_full[buf], (local / L::NBUF) & 1);
        tc_fence_after();
        for (int ly = 0; ly < S; ++ly) {
          const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + buf * L::TILE_COLS + ly * BN + col0;
          float* prow = reinterpret_cast<float*>(base + L::HALO_OFF) + (size_t)(ly * 128 + q * 32 + lane) * L::PSTRIDE + col0;
#pragma unroll 1
          for (int j = 0; j < EW / CH; ++j) {
            uint32_t r[CH];
            tmem_ld_32x32b<CH>(tbase + j * CH, r);
#pragma unroll
            for (int e = 0; e < CH; e += 4)
              *reinterpret_cast<float4*>(prow + j * CH + e) =
                  make_float4(__uint_as_float(r[e]), __uint_as_float(r[e + 1]), __uint_as_float(r[e + 2]),
                              __uint_as_float(r[e + 3]));
          }
        }
        continue;
      }
      const int c_base = (t % n_tiles) * BN + col0;
      const int nch = max(0, min(EW, p.n_out - c_base));
      const int pi = mt * P + pl;
      const bool valid = pi < count;
      // dense-masked channel schedule: this row's sample keeps / drops each channel
      const uint8_t* cmask = (p.ymask_channel && valid)
                                 ? p.ymask_channel + (size_t)(list_cell(p, pi) / (p.cells_h * p.cells_w)) * p.n_out
                                 : nullptr;
      mbar_wait(&acc_full[buf], (local / L::NBUF) & 1);
      tc_fence_after();
      for (int ly = 0; ly < S; ++ly) {
        const long long dst = (long long)pi * s2 + ly * S + lx;  // compact h2 row (patch-major)
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + buf * L::TILE_COLS + ly * BN + col0;
#pragma unroll 1
        for (int j = 0; j < EW / CH; ++j) {
          uint32_t r[CH];
          tmem_ld_32x32b<CH>(tbase + j * CH, r);
#pragma unroll
          for (int g = 0; g < CH / 8; ++g) {
            const int cl = j * CH + g * 8;
            float v[8];
            uint2 mk = make_uint2(0xffffffffu, 0xffffffffu);
            if (cmask && c_base + cl < p.n_out) mk = __ldg(reinterpret_cast<const uint2*>(cmask + c_base + cl));
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int c = c_base + cl + e;
              v[e] = fmaf(__uint_as_float(r[g * 8 + e]), vsc[c], vbi[c]);
              if (!(((e < 4 ? (mk.x >> (8 * e)) : (mk.y >> (8 * (e - 4)))) & 0xff))) v[e] = 0.f;
              if (p.relu) v[e] = fmaxf(v[e], 0.f);
            }
            uint4 w;
            w.x = pack_bf16x2(v[0], v[1]);
            w.y = pack_bf16x2(v[2], v[3]);
            w.z = pack_bf16x2(v[4], v[5]);
            w.w = pack_bf16x2(v[6], v[7]);
            *reinterpret_cast<uint4*>(stg + lane * L::STG_ROW + (cl >> 3) * 16) = w;
          }
        }
        if (ly == S - 1) {  // accumulators of this buffer consumed: hand back to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[buf]);
        }
        __syncwarp();
        // row-major sweep: each instruction writes 32 / CPR whole row slices
        constexpr int RPI = 32 / CPR;
        const int cc = lane % CPR, rr0 = lane / CPR;
#pragma unroll 4
        for (int it2 = 0; it2 < CPR; ++it2) {
          const int rw = it2 * RPI + rr0;
          const int rv = __shfl_sync(0xffffffffu, (int)valid, rw);
          const long long dr = __shfl_sync(0xffffffffu, dst, rw);
          if (rv && cc * 8 < nch)
            *reinterpret_cast<uint4*>(outp + dr * p.out_ld + c_base + cc * 8) =
                *reinterpret_cast<const uint4*>(stg + rw * L::STG_ROW + cc * 16);
        }
        __syncwarp();
      }
    }
  }

  if (KS > 1 || tail) {
    // split-K reduction through distributed shared memory: CTA ks finishes rows
    // [ks, ks + 1) * S*128/NP of its part tile's (ly, row) space, summing the NP
    // partials in rank order (deterministic), then scale / bias / ReLU -> bf16
    cluster_sync();  // every CTA's partials written and visible cluster-wide
    const int tr = KS > 1 ? (t_begin < tiles ? t_begin : -1) : split_t;
    if (tr >= 0) {
      const int mt = tr / n_tiles, n0 = (tr % n_tiles) * BN;
      constexpr int RR = S * 128;
      const int rpc = RR / NP;
      constexpr int C4 = BN / 4;
      const uint32_t partb = base_u32 + L::HALO_OFF;
      __nv_bfloat16* outp = reinterpret_cast<__nv_bfloat16*>(p.out);
      for (int idx = threadIdx.x; idx < rpc * C4; idx += THREADS) {
        const int lr = ks * rpc + idx / C4, c4 = idx % C4;
        const int ly = lr / 128, row = lr % 128;
        const int lx = row / P, pl = row - lx * P;
        const int pi = mt * P + pl;
        const int c = n0 + c4 * 4;
        if (pi >= count || c >= p.n_out) continue;
        const uint32_t off = (uint32_t)(((ly * 128 + row) * L::PSTRIDE + c4 * 4) * 4);
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int r = 0; r < NP; ++r) {
          float4 v;
          asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                       : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                       : "r"(mapa_shared(partb + off, r)) : "memory");
          acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        float o[4] = {acc.x, acc.y, acc.z, acc.w};
        uint32_t mk = 0xffffffffu;
        if (p.ymask_channel)
          mk = __ldg(reinterpret_cast<const uint32_t*>(
              p.ymask_channel + (size_t)(list_cell(p, pi) / (p.cells_h * p.cells_w)) * p.n_out + c));
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          o[e] = fmaf(o[e], vsc[c + e], vbi[c + e]);
          if (!((mk >> (8 * e)) & 0xff)) o[e] = 0.f;
          if (p.relu) o[e] = fmaxf(o[e], 0.f);
        }
        const long long dst = (long long)pi * s2 + ly * S + lx;
        *reinterpret_cast<uint2*>(outp + dst * p.out_ld + c) = make_uint2(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]));
      }
    }
    cluster_sync();  // peers done reading this CTA's partials
  }
  tc_fence_before();
  __syncthreads();
  if (warp == WARP_MMA) {
    tc_fence_after();
    tmem_dealloc<L::TMEM_COLS>(tmem_base);
  }
}

template <int S, int BN>
cudaError_t launch(const CUtensorMap& ta, const CUtensorMap& tb, const ConvParams& p, int num_sms,
                   cudaStream_t stream) {
  using L = Cfg<S, BN>;
  auto kern = patch_conv_kernel<S, BN>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::ALLOC);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int s2 = S * S;
  const long long tiles = ((long long)(p.rows_max / s2) + L::P - 1) / L::P * ((p.n_out + BN - 1) / BN);
  if ((p.ksplit > 1 || p.tail_split) && L::SPLIT_OK) {  // clusters (host-checked)
    // ksplit: one wave of clusters, one tile each; tail split: a persistent grid
    // of 2-CTA clusters
    const long long g = p.ksplit > 1 ? tiles * p.ksplit : (tiles < num_sms ? tiles : num_sms) / 2 * 2;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(g > 2 ? g : 2), 1, 1);
    cfg.blockDim = dim3(THREADS, 1, 1);
    cfg.dynamicSmemBytes = L::ALLOC;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = p.ksplit > 1 ? p.ksplit : 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, kern, ta, tb, p);
  }
  int grid = (int)(tiles < num_sms ? tiles : num_sms);
  if (grid < 1) grid = 1;
  return launch_k(kern, dim3(grid), dim3(THREADS), L::ALLOC, stream, ta, tb, p);
}

}  // namespace pc

// Host dispatch (capi.cu): S in {2, 4}, stride 1, 3x3, n_out <= 512.
bool patch_conv_supported(int s, int bn) {
  return (s == 2 && (bn == 128 || bn == 64)) || (s == 4 && (bn == 64 || bn == 128));
}

cudaError_t launch_patch_conv(const CUtensorMap& ta, const CUtensorMap& tb, const ConvParams& p, int s, int bn,
                              int num_sms, cudaStream_t stream) {
  if (s == 2 && bn == 128) return pc::launch<2, 128>(ta, tb, p, num_sms, stream);
  if (s == 2 && bn == 64) return pc::launch<2, 64>(ta, tb, p, num_sms, stream);
  if (s == 4 && bn == 64) return pc::launch<4, 64>(ta, tb, p, num_sms, stream);
  if (s == 4 && bn == 128) return pc::launch<4, 128>(ta, tb, p, num_sms, stream);
  return cudaErrorInvalidValue;
}

}  // namespace laud
