// Conv engine dispatch: tile width / pair / A mode / epilogue mode -> the
// instantiation compiled in conv_gemm_bn*.cu (kernel: conv_gemm.cuh).
#include "conv_gemm.cuh"

namespace laud {

cudaError_t launch_conv_gemm(const CUtensorMap& tmap_a, const CUtensorMap& tmap, const CUtensorMap& tmap_o, int bn,
                             const ConvParams& p, int num_sms, cudaStream_t stream, int pair) {
  const int n_tiles = (p.n_out + bn - 1) / bn;
  ConvLaunch c;
  c.tmap_a = &tmap_a;
  c.tmap_b = &tmap;
  c.tmap_o = &tmap_o;
  c.p = &p;
  c.num_sms = num_sms;
  c.stream = stream;
  // EP_PLAIN*: bf16 out, no per-channel scale / coarse mask / masker-dot, bias
  // vector fits the smem cache (VEC_CACHE_FLOATS)
  // (a partial last N tile is fine — its extra columns are never stored —
  // except under the per-sample channel mask, read per column)
  const int npad = n_tiles * bn;
  c.ep_plain = !p.out_f32 && !p.scale && !p.col_index && !p.ymask_coarse && !p.mdot_w &&
               npad <= VEC_CACHE_FLOATS && (p.n_out % bn == 0 || !p.ymask_channel) &&
               (!p.adot_out || npad + p.kpad <= VEC_CACHE_FLOATS);  // + masker weights in smem
  c.relu_all = p.relu && !p.relu_inactive_coarse;
  if (p.ksplit > 1 && (!c.ep_plain || pair || p.adot_out || p.ymask_channel || p.relu_inactive_coarse))
    return cudaErrorInvalidValue;  // split-K runs only the plain epilogues (host-checked)
  c.am = p.a_tile ? (p.adot_out ? AM_TILE_DOT : AM_TILE) : p.a_box ? AM_BOX : p.a_tma ? AM_G4 : AM_ANY;
  if (pair) {
    if (bn != 256) return cudaErrorInvalidValue;
    c.tiles_max = ((p.rows_max + 2 * BM - 1) / (2 * BM)) * n_tiles;
    return launch_conv_pair(c, pair);
  }
  c.tiles_max = ((p.rows_max + BM - 1) / BM) * n_tiles;
  switch (bn) {
    case 64: return launch_conv_bn64(c);
    case 128: return launch_conv_bn128(c);
    case 256: return launch_conv_bn256(c);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace laud
