// Conv engine instantiations for CTA-pair (cta_group::2) 256 x 256 tiles.
#include "conv_gemm.cuh"

namespace laud {
// pair = 1: 4 operand stages; pair = 2: short K, 2 stages and double-buffered
// epilogue staging.  The B tensor map's box is BN / 2 rows (each CTA loads half).
cudaError_t launch_conv_pair(const ConvLaunch& c, int pair) {
  const ConvParams& p = *c.p;
  if (!p.a_tile || p.adot_out) return cudaErrorInvalidValue;  // pairs: TMA-box A rows, no masker readers
  if (pair == 2)
    return !c.ep_plain ? launch_bn<256, 2, 2, true, AM_TILE, EP_ANY>(*c.tmap_a, *c.tmap_b, *c.tmap_o, p, c.tiles_max, c.num_sms, c.stream)
           : p.resid   ? launch_bn<256, 2, 2, true, AM_TILE, EP_PLAIN_RES>(*c.tmap_a, *c.tmap_b, *c.tmap_o, p, c.tiles_max, c.num_sms, c.stream)
                       : launch_bn<256, 2, 2, true, AM_TILE, EP_PLAIN>(*c.tmap_a, *c.tmap_b, *c.tmap_o, p, c.tiles_max, c.num_sms, c.stream);
  return !c.ep_plain ? launch_bn<256, 4, 1, true, AM_TILE, EP_ANY>(*c.tmap_a, *c.tmap_b, *c.tmap_o, p, c.tiles_max, c.num_sms, c.stream)
         : p.resid   ? launch_bn<256, 4, 1, true, AM_TILE, EP_PLAIN_RES>(*c.tmap_a, *c.tmap_b, *c.tmap_o, p, c.tiles_max, c.num_sms, c.stream)
                     : launch_bn<256, 4, 1, true, AM_TILE, EP_PLAIN>(*c.tmap_a, *c.tmap_b, *c.tmap_o, p, c.tiles_max, c.num_sms, c.stream);
}
}  // namespace laud
