/* laud.h — C-ABI of the B200 LAUDNet dynamic-inference path.
 *
 * One shared library (paper_2308_15949_b200/_laud.so, sm_100a) behind the
 * Python operator surface of the reference's `dynlat.reference`.  Plain
 * pointers and sizes only; every device pointer is caller-allocated CUDA
 * memory, every call is stream-ordered and asynchronous (no host sync, no
 * allocation on the hot path), `stream` is a cudaStream_t (NULL = legacy).
 *
 * Layout: activations NHWC bfloat16 with a per-pixel channel stride `ld`
 * (multiple of 8, channels zero-padded); weights packed bf16
 * [c_out][k*k taps][kpad(c_in)] (kpad = c_in rounded up to 64, zero filled);
 * folded-BN scale/bias fp32 [c_out] (NULL = 1 / 0); masks uint8 per cell,
 * active-cell and active-pixel lists int32 row-major (n, i, j) linear index.
 *
 * Status codes map onto the reference's exception classes
 * (`pkg/src/dynlat/errors.py:8-29`); the Python layer re-raises them.
 */
#ifndef LAUD_H_
#define LAUD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LAUD_OK 0
#define LAUD_ERR_GRANULARITY 1 /* GranularityMismatch (reference.py:171-172, 304-305) */
#define LAUD_ERR_MASK_SHAPE 2  /* MaskShapeMismatch (reference.py:307-310, 332-335)  */
#define LAUD_ERR_SHAPE 3       /* ShapeMismatch (reference.py:36-37, 54-67)           */
#define LAUD_ERR_UNSUPPORTED 4 /* ShapeMismatch: channel skipping with groups != 1 (reference.py:405-406) */
#define LAUD_ERR_CUDA 5        /* launch / runtime failure                            */
#define LAUD_ERR_ARG 6         /* ValueError: bad argument                            */

#define LAUD_PARADIGM_SPATIAL 0
#define LAUD_PARADIGM_CHANNEL 1
#define LAUD_PARADIGM_LAYER 2
#define LAUD_PARADIGM_STATIC 3

/* Library identity and the calling thread's last error message. */
const char* laud_version(void);
const char* laud_last_error(void);
/* Number of kernels this library launched since load (diagnostics / bench). */
uint64_t laud_launch_count(void);

/* Per-launch CUDA-event profiling (off by default; outside timed regions).
 * laud_profile_end synchronises, fills up to max_records records in launch
 * order and returns how many were written.  rows = actual GEMM rows (device
 * count resolved), k = kernel taps * input channels; flops = 2*rows*n_out*k. */
typedef struct laud_profile_record {
  int tag; /* 0 conv engine, 1 masker, 2 compaction/dilation, 3 glue */
  float ms;
  long long rows, n_out, k, bytes;
  int taps, resid; /* conv: kernel taps, residual read in the epilogue */
} laud_profile_record;
void laud_profile_begin(void);
int laud_profile_end(laud_profile_record* out, int max_records);

/* Bytes of look-back scratch for a compaction over `items` elements.  Must be
 * zeroed once after allocation; the kernels restore it to zero. */
size_t laud_scan_workspace_bytes(int items);
/* fp32 partial sums the spatial masker needs for this geometry. */
size_t laud_masker_partial_floats(int n, int h, int w, int c, int s, int stride);

/* Spatial (and layer, s*stride = H) masker — replaces
 * `spatial_masker_forward` + `build_gather_plan` (reference.py:156-186, 133-135)
 * with the fused-masker identity of reference.py:244-253: decision per cell of
 * the OUTPUT grid = mean over the (s*stride)^2 input window of x.wdiff + bias
 * >= 0 (x bf16, or fp32 when x_f32).  Writes coarse[n*(H/(s*st))*(W/(s*st))], the row-major list of active
 * cells and its device-side count. */
int laud_spatial_masker(const void* x, int x_f32, int ld, int n, int h, int w, int c, int s,
                        int stride, const float* wdiff, float bias, uint8_t* coarse,
                        int* cell_list, int* cell_count, float* partial, void* scan,
                        void* stream);

/* Active-cell list from a caller-supplied coarse mask (argwhere order). */
int laud_cells_from_mask(const uint8_t* coarse, int cells, int* cell_list, int* cell_count,
                         void* scan, void* stream);

/* conv1 work set: input pixels covered by an active cell's window grown by
 * `radius` (1 = conv2's 3x3 halo).  With stride 1 this is exactly the
 * Chebyshev dilation of reference.py:226-241 (`dilate_and_rates`, k = 2r+1). */
int laud_dilate_pixels(const uint8_t* coarse, int n, int h_in, int w_in, int s, int stride,
                       int radius, int* pix_list, int* pix_count, void* scan, void* stream);

/* Generic implicit-GEMM convolution (tcgen05 / TMEM / TMA engine). */
typedef struct laud_conv_args {
  int row_mode; /* 0 dense output grid, 1 active-patch list, 2 pixel list */
  const int* list;
  const int* count; /* device count, NULL -> rows_max */
  int rows_max;
  int batch, out_h, out_w;
  int patch_h, patch_w, cells_h, cells_w;
  const void* act;
  int in_h, in_w, in_c, in_ld;
  int a_compact;
  int ksize, stride, pad;
  const void* weight; /* packed [n_out][ksize*ksize][kpad(in_c) (+64 grouped)] bf16 */
  int n_out;
  const float* scale;
  const float* bias;
  int relu;
  int out_mode; /* 0 scatter to output pixel, 1 compact row */
  void* out;
  int out_ld;
  int out_f32;
  const void* resid;
  int resid_ld;
  const uint8_t* relu_inactive_coarse;
  const uint8_t* ymask_coarse;  /* dense-masked: y *= coarse[cell]       */
  const uint8_t* ymask_channel; /* dense-masked: y *= mask[n][channel]   */
  /* per-sample dynamic width (channel skipping): rows padded per sample to
   * sample_rows (multiple of 128); k_n = chan_count[n]; n_dyn skips output
   * columns >= k_n, k_dyn runs K = taps * roundup(k_n, 64); b_batched: weight
   * is [batch][n_out][K]; col_index[n][col_index_ld] maps output column ->
   * scale/bias channel. */
  int sample_rows;
  const int* chan_count;
  int n_dyn, k_dyn, b_batched;
  const int* col_index;
  int col_index_ld;
  /* masker-conv3 fusion: per output row, dot(stored output, mdot_w) is added
   * into mdot_out[cell of the row] (patch rows) — the next block's masker. */
  const float* mdot_w;
  float* mdot_out;
  int misplace_first;
  /* grouped convolution (RegNet conv2): groups > 1 with in_c / groups and
   * n_out / groups channels per group (in_c / groups a multiple of 8); the
   * weight is the dense block-diagonal [n_out][taps][kpad(in_c) + 64] (zeros
   * outside the group; the extra 64 zero columns let an output tile's K
   * window run past the last group).  0 or 1 = dense. */
  int groups;
  /* fp32 mode: act / weight / resid / out are fp32 (weight in the same packed
   * layout), computed with fp32 FFMA (the 1e-5 numerics path). */
  int fp32;
  /* per-sample weights gathered in the kernel (channel skipping at large
   * batch, needs sample_rows + chan_count): b_gather = 1 -> B rows are weight
   * rows b_index[n][j] for output columns j < k_n (weight packed as usual);
   * b_gather = 2 -> weight is
   * the TRANSPOSED 1x1 kernel [K rows][n_out] and the tile's K rows are
   * b_index[n][k], k < k_n (compact A of k_n channels).  b_rows: rows of the
   * gathered weight tensor.  0 = packed / batched B as above. */
  int b_gather;
  const int* b_index;
  int b_index_ld;
  int b_rows;
  /* small grids: the halo patch conv (3x3 over S x S patches) may split K over
   * a thread-block cluster (fp32 partials reduced through distributed shared
   * memory) when one wave of tiles leaves SMs idle — a different fp32
   * summation order than the unsplit conv, so off by default (the mirror API
   * keeps sparse == dense-masked bitwise); the network executor enables it. */
  int latency_split;
  /* > 1 (ROWS_PATCH): each list entry e stands for the list_expand cells
   * e*k .. e*k+k-1 (k = list_expand) and the device count scales by k — a
   * layer block's active-sample list read as its samples' S x S cells. */
  int list_expand;
} laud_conv_args;

int laud_conv(const laud_conv_args* a, void* stream);

/* Debug only (tools/engine_trace.py): when dev_buf (16384 u64, device) is set,
 * CTA 0 of every following conv launch records %globaltimer at its pipeline
 * events; NULL turns it off.  Not for use on a timed path. */
void laud_debug_set_trace(void* dev_buf);

/* One bottleneck block forward — replaces `block_forward_sparse`
 * (reference.py:356-436) for SPATIAL / LAYER / STATIC.  Masks: either
 * given (`given_coarse`, uint8 per cell; spatial cells on the output grid,
 * layer = one per sample) or computed by the masker (`masker_wdiff`,
 * `masker_bias`).  `out` may alias `x` only when the block has no
 * downsample and shapes match (in-place residual). */
typedef struct laud_block_args {
  int paradigm;
  int n, h_in, w_in, c_in, x_ld;
  int c_mid, c_out, stride, groups;
  int s; /* spatial granularity S (output grid) */
  int has_down;
  const void* x;
  void* out;
  const void* w1;
  const void* w2;
  const void* w3;
  const void* wd;
  const float *s1, *b1, *s2, *b2, *s3, *b3, *sd, *bd;
  int relu1, relu2, relu_out;
  const float* masker_wdiff;
  float masker_bias;
  const uint8_t* given_coarse;
  /* outputs + workspace (laud_block_workspace_bytes) */
  uint8_t* coarse_out;
  int* cell_list;
  int* cell_count;
  int* pix_list;
  int* pix_count;
  void* h1;
  void* h2;
  float* partial;
  void* scan;
  int misplace_first; /* test-only fault hook (reference.py:362, 400-401) */
  /* channel paradigm (reference.py:189-218, 404-423): masker MLP weights
   * fp32 w1 [hidden][c_in], w2 [2D][hidden]; G channels per decision; either
   * a given expanded mask [n][c_mid] (uint8) or the masker runs.  Outputs:
   * coarse [n][D], expanded [n][c_mid], kept lists sel [n][c_mid] + count [n],
   * optional logit gaps dvals [n][D]; wpack = laud_channel_pack_bytes(). */
  const float* ch_w1;
  const float* ch_w2;
  int ch_hidden, ch_d, ch_groups;
  const uint8_t* given_chmask;
  uint8_t* ch_coarse;
  uint8_t* ch_expanded;
  int* ch_sel;
  int* ch_count;
  float* ch_dvals;
  void* wpack;
  /* masker-conv3 fusion across consecutive blocks of a stage (same grid, S):
   * dn [cells] carries, for cells prev_coarse marks active, the dot product of
   * this block's input with its masker weights (accumulated by the previous
   * block's conv3 epilogue); cells it skipped are read from x.  When
   * next_wdiff is set, this block's conv3 accumulates the dots for the next
   * block into dn (the masker zeroes dn first). */
  const uint8_t* prev_coarse;
  float* dn;
  const float* next_wdiff;
  /* EXT: per-decision bias added to the channel masker's logit gap l0 - l1
   * (nullable; calibrates the kept ratio like a trained FLOPs loss would). */
  const float* ch_bias;
  /* fp32 mode: x / out / h1 / h2 fp32 and fp32 weights (same packed layouts);
   * every conv on the fp32 FFMA engine (1e-5 numerics path). */
  int fp32;
  /* spatial: run conv1 densely on the input grid (the reference's own
   * schedule, reference.py:385) instead of on the dilated pixel list — cheaper
   * when the dilated set covers most pixels (S <= 2 at ratio >= 0.4). */
  int conv1_dense;
  /* EXT squeeze-excitation after conv2 (RegNetY; se_hidden = C_mid / se_reduction,
   * reference core.py:195): per sample, gate = sigmoid(se_w2 relu(se_w1 mean(h2)
   * + se_b1) + se_b2) over the sample's conv2 rows (its active patches under a
   * spatial mask), h2 *= gate.  fp32 [se_hidden][c_mid], [se_hidden], [c_mid][se_hidden],
   * [c_mid]; se_w1 NULL = no SE (the reference executor has none). */
  const float* se_w1;
  const float* se_b1;
  const float* se_w2;
  const float* se_b2;
  int se_hidden;
  /* spatial masker fused into a dense conv1 (conv1_dense, masker computed):
   * scratch for one masker dot per conv1 input pixel [n * h_in * w_in] fp32,
   * written (not accumulated) by conv1's readers and summed per cell in a
   * fixed order by the decision pass, so decisions are deterministic;
   * NULL = standalone masker pass. */
  float* cell_sums;
  /* EXT channel skipping over a grouped conv2 (RegNet; the reference's sparse
   * executor rejects groups != 1, reference.py:405-406): the grouped kernel
   * expanded block-diagonally to a dense [c_mid][9][kpad] kernel, so the
   * per-sample schedule's W2[sel][:, sel] keeps each group's kept links — the
   * sparse form of the reference's dense-masked channel forward
   * (reference.py:331-339); w2 keeps the grouped layout, which the
   * dense-masked schedule uses.  NULL = the reference behaviour
   * (LAUD_ERR_UNSUPPORTED for groups != 1). */
  const void* w2_dense;
  /* channel paradigm at batch >= 8: conv3's kernel transposed, bf16
   * [c_mid][c_out] (K rows, c_out contiguous), for the in-kernel K gather
   * W3[:, sel] (conv2's N gather W2[sel] uses w2).  NULL = dense-masked
   * schedule at large batch. */
  const void* w3t;
  /* optional second stream: at small grids (<= 4096 mask cells) the spatial /
   * layer masker runs there, concurrently with conv1 (both only read x), and
   * the block's stream waits for it before the skip path and conv2 (graph
   * capture: a fork/join).  NULL = masker on `stream` (or fused into conv1). */
  void* aux_stream;
  /* allow the conv2 split-K of laud_conv_args.latency_split at small grids. */
  int latency_split;
} laud_block_args;

/* Channel masker alone — replaces `channel_masker_forward` (reference.py:189-218):
 * GAP over hw pixels, relu(w1 gap), w2 hidden -> d interleaved pairs, keep iff
 * l0 >= l1, G-fold expansion to cm (= d*g) channels padded to cm_p, ordered
 * kept-channel lists sel [n][cm_p] and counts [n]; dvals = l0 - l1 (nullable). */
int laud_channel_masker(const void* x, int x_f32, int ld, int n, int hw, int c, const float* w1,
                        int hidden, const float* w2, int d, int g, int cm, int cm_p,
                        uint8_t* coarse, float* dvals, uint8_t* expanded, int* sel, int* count,
                        const float* bias, void* stream);

/* Bytes of per-sample packed weights the channel paradigm needs. */
size_t laud_channel_pack_bytes(int n, int c_in, int c_mid, int c_out);

int laud_block_forward(const laud_block_args* a, void* stream);

/* Network glue: stem im2col from uint8 NHWC images (mean/std normalised),
 * 3x3/s2 max-pool, global average pool. */
int laud_stem_im2col(const uint8_t* img, int n, int h, int w, int k, int stride, int pad,
                     const float* mean, const float* inv_std, void* cols, int cols_ld,
                     void* stream);
int laud_maxpool3s2(const void* x, int n, int h, int w, int c, void* y, void* stream);
/* Fused ResNet stem: uint8 NHWC 224x224x3 images -> (normalise, 7x7/2 conv,
 * + bias, ReLU, 3x3/2 max-pool) -> bf16 NHWC [n][56][56][64], one kernel (no
 * im2col in HBM).  weight: bf16 [64][256], K index ky*32 + kx*4 + c (kx < 7,
 * c < 3; other entries zero); bias fp32 [64]. */
int laud_stem_pool(const uint8_t* img, int n, int h, int w, const float* mean, const float* inv_std,
                   const void* weight, const float* bias, void* out, void* stream);
/* Fused RegNet stem: uint8 NHWC 224x224x3 images -> (normalise, 3x3/2 conv,
 * + bias, ReLU) -> bf16 NHWC [n][112][112][32], one kernel (no im2col).
 * weight: bf16 [32][3][16], K index kx*4 + c (kx < 3, c < 3; others zero). */
int laud_stem3(const uint8_t* img, int n, int h, int w, const float* mean, const float* inv_std,
               const void* weight, const float* bias, void* out, void* stream);
int laud_global_avgpool(const void* x, int n, int hw, int c, void* y, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LAUD_H_ */
