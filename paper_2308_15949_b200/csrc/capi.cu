// C-ABI of the LAUDNet B200 path (include/laud.h): argument validation with
// the reference's error taxonomy, TMA descriptor cache, and the block-level
// composition of masker -> dilate -> gather-conv1 -> patch conv2 ->
// conv3 + scatter-add (reference semantics `reference.py:356-436`).
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/laud.h"
#include "laud_conv.cuh"

namespace laud {
cudaError_t launch_conv_gemm(const CUtensorMap& tmap_a, const CUtensorMap& tmap, const CUtensorMap& tmap_o, int bn,
                             const ConvParams& p, int num_sms, cudaStream_t stream, int pair);
cudaError_t launch_conv_f32(const ConvParams& p, cudaStream_t stream);
bool patch_conv_supported(int s, int bn);
cudaError_t launch_patch_conv(const CUtensorMap& ta, const CUtensorMap& tb, const ConvParams& p, int s, int bn,
                              int num_sms, cudaStream_t stream);
size_t scan_state_bytes(int total);
int masker_splits(int win, int c, int* chunks_per_split);
cudaError_t launch_spatial_masker(const void* x, int x_f32, int ld, int n, int h, int w, int c,
                                  int s, int stride, const float* wdiff, float bias,
                                  uint8_t* coarse, int* list, int* count, float* partial,
                                  void* scan, cudaStream_t stream, const uint8_t* prev_coarse,
                                  float* dn);
cudaError_t launch_list_from_mask(const uint8_t* coarse, int total, int* list, int* count,
                                  void* scan, cudaStream_t stream);
cudaError_t launch_masker_decide(const float* pixel_dots, int n, int h, int w, int win, float bias,
                                 uint8_t* coarse, int* list, int* count, void* scan, cudaStream_t stream);
cudaError_t launch_dilate_pixels(const uint8_t* coarse, int n, int h, int w, int s, int stride,
                                 int cells_h, int cells_w, int radius, int* list, int* count,
                                 void* scan, cudaStream_t stream);
cudaError_t launch_se_channel(void* h2, int n, int c, int hw, int sr, const int* sel, const int* count,
                              const float* w1, const float* b1, int hs, const float* w2, const float* b2,
                              void* scratch, cudaStream_t s);
cudaError_t launch_stem_im2col(const uint8_t* img, int n, int h, int w, int k, int stride, int pad,
                               const float* mean, const float* inv_std, void* cols, int cols_ld,
                               cudaStream_t s);
cudaError_t launch_maxpool3s2(const void* x, int n, int h, int w, int c, void* y, cudaStream_t s);
cudaError_t launch_gap(const void* x, int n, int hw, int c, void* y, cudaStream_t s);
cudaError_t launch_stem3(const uint8_t* img, int n, const float* mean, const float* inv_std, const void* wpk,
                         const float* bias, void* out, int num_sms, cudaStream_t s);
cudaError_t launch_stem_pool(const uint8_t* img, int n, const float* mean, const float* inv_std,
                             const void* wpk, const float* bias, void* out, int num_sms, cudaStream_t s);
cudaError_t launch_se(void* h2, int n, int c, const int* list, const int* count, int cells_per_img,
                      int rows_per_cell, int rows_per_img, const float* w1, const float* b1, int hs,
                      const float* w2, const float* b2, void* scratch, cudaStream_t s);
cudaError_t launch_channel_masker(const void* x, int x_f32, int ld, int n, int hw, int c,
                                  const float* w1, int hd, const float* w2, int d, int g, int cm,
                                  int cm_p, uint8_t* coarse, float* dvals, uint8_t* expanded,
                                  int* sel, int* count, const float* bias, cudaStream_t s);
cudaError_t launch_channel_lists(const uint8_t* expanded, int n, int cm_p, int* sel, int* count,
                                 cudaStream_t s);
cudaError_t launch_pack_weights(const void* src, int src_rows, int taps, int src_k, void* dst,
                                int dst_rows, int dst_k, const int* sel, const int* count,
                                int sel_ld, int row_sel, int col_sel, int n, cudaStream_t s);
}  // namespace laud

using namespace laud;

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};
unsigned long long* g_trace = nullptr;  // laud_debug_set_trace (tools only)

// Optional per-launch CUDA-event profiling (laud_profile_*), off by default.
struct ProfRec {
  int tag;               // 0 conv, 1 masker, 2 compaction/dilate, 3 glue
  cudaEvent_t e0, e1;
  int snap;              // index of the count snapshot (-1: none)
  long long rows_per_count, rows_max, n_out, k_alg, bytes;
  int taps, resid;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
int* g_prof_counts = nullptr;  // device snapshots of row counts at launch time
int g_prof_nsnap = 0;
constexpr int kProfSnaps = 8192;

struct ProfScope {
  ProfRec rec;
  bool on;
  cudaStream_t st;
  ProfScope(int tag, cudaStream_t s, const int* count = nullptr) : on(false), st(s) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (!g_prof_on) return;
    on = true;
    memset(&rec, 0, sizeof(rec));
    rec.tag = tag;
    rec.snap = -1;
    if (count && g_prof_counts && g_prof_nsnap < kProfSnaps) {  // snapshot before e0
      rec.snap = g_prof_nsnap++;
      cudaMemcpyAsync(g_prof_counts + rec.snap, count, sizeof(int), cudaMemcpyDeviceToDevice, st);
    }
    cudaEventCreate(&rec.e0);
    cudaEventCreate(&rec.e1);
    cudaEventRecord(rec.e0, st);
  }
  ~ProfScope() {
    if (!on) return;
    cudaEventRecord(rec.e1, st);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.push_back(rec);
  }
};

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_check(cudaError_t e, const char* what, int launches) {
  if (e != cudaSuccess) return fail(LAUD_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  g_launches += launches;
  return LAUD_OK;
}

int round_up(int v, int m) { return (v + m - 1) / m * m; }

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 148;
  }
  return cached[dev];
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

struct MapKey {
  const void* ptr;
  int rows, k, bn, dev;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && rows == o.rows && k == o.k && bn == o.bn && dev == o.dev;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    return std::hash<const void*>()(k.ptr) ^ ((size_t)k.rows << 1) ^ ((size_t)k.k << 21) ^
           ((size_t)k.bn << 41) ^ ((size_t)k.dev << 50);
  }
};

std::mutex g_map_mu;
std::unordered_map<MapKey, CUtensorMap, MapKeyHash> g_maps;

// Weights [rows][k] bf16, k contiguous; box = 64 (k) x bn (rows), 128B swizzle,
// rows past the end read as zeros.
int tensor_map_2d(const void* w, int rows, int k, int ld, int bn, CUtensorMap* out,
                  int batch = 0) {
  int dev = 0;
  cudaGetDevice(&dev);
  MapKey key{w, rows + batch * 1000003, k * 65536 + ld, bn, dev};
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return LAUD_OK;
    }
  }
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(LAUD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(w) & 15) != 0)
    return fail(LAUD_ERR_ARG, "weight pointer must be 16-byte aligned");
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)k, (cuuint64_t)rows, (cuuint64_t)(batch > 0 ? batch : 1)};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 2, (cuuint64_t)ld * 2 * rows};
  cuuint32_t box[3] = {64, (cuuint32_t)bn, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, batch > 0 ? 3 : 2, const_cast<void*>(w),
                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LAUD_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    g_maps[key] = m;
  }
  *out = m;
  return LAUD_OK;
}

// Activation as a 4D tensor [batch][h][w][c] (c contiguous, row stride ld) with a
// {64 ch, S, S, 1} box traversed at the conv stride: one TMA op loads one S x S
// patch's tap window (OOB -> zeros, negative coordinates included).
int tensor_map_patch(const void* act, int batch, int h, int w, int c, int ld, int s, int stride,
                     CUtensorMap* out) {
  int dev = 0;
  cudaGetDevice(&dev);
  MapKey key{act, -(batch * 4096 + h), -(w * 65536 + c), -(ld * 64 + s * 8 + stride), dev};
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return LAUD_OK;
    }
  }
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                               CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                               CUtensorMapFloatOOBfill);
  EncodeFn fn = reinterpret_cast<EncodeFn>(encode_fn());
  if (!fn) return fail(LAUD_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMap m;
  cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)batch};
  cuuint64_t strides[3] = {(cuuint64_t)ld * 2, (cuuint64_t)w * ld * 2, (cuuint64_t)h * w * ld * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)(s * stride), (cuuint32_t)(s * stride), 1};
  cuuint32_t estr[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(act), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(LAUD_ERR_CUDA, "cuTensorMapEncodeTiled (patch box) failed (%d)", (int)r);
  {
    std::lock_guard<std::mutex> lk(g_map_mu);
    g_maps[key] = m;
  }
  *out = m;
  return LAUD_OK;
}

// Tile width: BN=128 (double-buffered epilogue staging) for epilogue-heavy
// small-K convs and for grids too small to fill the SMs at BN=256.
int pick_bn(int n_out, int k, long long rows) {
  static const int forced = [] {
    const char* e = getenv("LAUD_BN");
    return e ? atoi(e) : 0;
  }();
  if (forced == 64 || forced == 128 || forced == 256) return n_out <= 64 ? 64 : forced;
  if (n_out <= 64) return 64;
  // grids under one wave (small batch): narrower N tiles give more CTAs, each
  // with a shorter B stream — the single-CTA K loop is the latency there
  static const int small_env = [] {
    const char* e = getenv("LAUD_SMALL_GRID_BN");
    return e ? atoi(e) : 1;
  }();
  const long long mt = (rows + 127) / 128;
  if (small_env && mt * ((n_out + 63) / 64) <= num_sms()) return 64;
  if (small_env && mt * ((n_out + 127) / 128) <= num_sms()) return 128;
  if (n_out <= 128) return 128;
  // widths that 256-wide tiles pad badly (RegNet 336: 512 computed columns vs
  // 384 with 128-wide tiles) take 128-wide tiles
  const int pad256 = (n_out + 255) / 256 * 256, pad128 = (n_out + 127) / 128 * 128;
  if ((pad256 - pad128) * 10 > n_out) return 128;
  return 256;  // measured best for every R101 conv shape at batch 256 (tools/sweep_cfg.sh)
}

// Events of the block forward's masker fork/join (laud_block_args.aux_stream);
// reused call after call (stream-ordered, and under graph capture each record
// / wait pair becomes a graph edge at capture time).
cudaEvent_t fork_event(int i) {
  static cudaEvent_t ev[2] = {nullptr, nullptr};
  static std::once_flag once;
  std::call_once(once, [] {
    for (auto& e : ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  });
  return ev[i];
}

// Device list 0, 1, ..., items-1 (every cell of a grid active), built once per
// length outside graph capture and cached; nullptr when it would have to be
// allocated during a capture (the caller then keeps its dense schedule).
const int* identity_list(int items, cudaStream_t st) {
  static std::mutex mu;
  static std::unordered_map<long long, int*> lists;
  int dev = 0;
  cudaGetDevice(&dev);
  const long long key = ((long long)dev << 40) | (long long)items;
  std::lock_guard<std::mutex> lk(mu);
  auto it = lists.find(key);
  if (it != lists.end()) return it->second;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
  std::vector<int> h(items);
  for (int i = 0; i < items; ++i) h[i] = i;
  int* d = nullptr;
  if (cudaMalloc(&d, (size_t)items * sizeof(int)) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, h.data(), (size_t)items * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return nullptr;
  }
  lists[key] = d;
  return d;
}

// fused masker dots riding on a dense 1x1 conv (ConvParams::adot_*)
struct AdotArgs {
  const float* w;
  float* out;  // one dot per dense row (input pixel)
};
constexpr int LAUD_ADOT_UNAVAILABLE = 99;  // internal: conv shape cannot host the masker

int run_conv(const laud_conv_args* a, cudaStream_t st, const AdotArgs* ad = nullptr) {
  if (!a || !a->act || !a->weight || !a->out) return fail(LAUD_ERR_ARG, "null pointer in conv args");
  if (a->in_c % 8 || a->in_ld % 8 || a->in_ld < a->in_c)
    return fail(LAUD_ERR_SHAPE, "in_c (%d) and in_ld (%d) must be multiples of 8, ld >= c", a->in_c,
                a->in_ld);
  if (a->n_out % 8 || a->out_ld % 8 || a->n_out < 8)
    return fail(LAUD_ERR_SHAPE, "n_out (%d) / out_ld (%d) must be multiples of 8", a->n_out,
                a->out_ld);
  if (a->ksize < 1 || a->ksize % 2 == 0) return fail(LAUD_ERR_ARG, "ksize must be odd");
  if (a->a_compact && a->ksize != 1) return fail(LAUD_ERR_ARG, "compact A needs a 1x1 kernel");
  if (a->row_mode != ROWS_DENSE && !a->list)
    return fail(LAUD_ERR_ARG, "row list required for patch/pixel rows");
  if (a->row_mode == ROWS_PATCH && (a->patch_h < 1 || a->patch_w < 1))
    return fail(LAUD_ERR_GRANULARITY, "patch size must be positive");
  if (a->rows_max <= 0) return LAUD_OK;
  ConvParams p;
  memset(&p, 0, sizeof(p));
  p.row_mode = a->row_mode;
  p.list = a->list;
  p.count = a->count;
  p.rows_max = a->rows_max;
  p.batch = a->batch;
  p.out_h = a->out_h;
  p.out_w = a->out_w;
  p.patch_h = a->patch_h > 0 ? a->patch_h : 1;
  p.patch_w = a->patch_w > 0 ? a->patch_w : 1;
  p.cells_h = a->cells_h > 0 ? a->cells_h : 1;
  p.cells_w = a->cells_w > 0 ? a->cells_w : 1;
  p.act = a->act;
  p.in_h = a->in_h;
  p.in_w = a->in_w;
  p.in_c = a->in_c;
  p.in_ld = a->in_ld;
  p.a_compact = a->a_compact;
  p.ksize = a->ksize;
  p.stride = a->stride;
  p.pad = a->pad;
  p.groups = a->groups > 1 ? a->groups : 1;
  if (p.groups > 1) {
    if (a->in_c % p.groups || a->n_out % p.groups || (a->in_c / p.groups) % 8)
      return fail(LAUD_ERR_SHAPE, "grouped conv: in_c (%d) / n_out (%d) must split into %d groups "
                  "of multiples of 8 input channels", a->in_c, a->n_out, p.groups);
    if (a->a_compact || a->sample_rows || a->chan_count)
      return fail(LAUD_ERR_UNSUPPORTED, "grouped conv: no compact / per-sample modes");
    p.gw_in = a->in_c / p.groups;
    p.gw_out = a->n_out / p.groups;
  }
  p.kpad = round_up(a->in_c, 64) + (p.groups > 1 ? 64 : 0);
  p.num_kb = a->ksize * a->ksize * p.kpad / 64;
  p.n_out = a->n_out;
  p.scale = a->scale;
  p.bias = a->bias;
  p.relu = a->relu;
  p.out_mode = a->out_mode;
  p.out = a->out;
  p.out_ld = a->out_ld;
  p.out_f32 = a->out_f32;
  p.resid = a->resid;
  p.resid_ld = a->resid_ld;
  p.relu_inactive_coarse = a->relu_inactive_coarse;
  p.ymask_coarse = a->ymask_coarse;
  p.ymask_channel = a->ymask_channel;
  p.sample_rows = a->sample_rows;
  p.chan_count = a->chan_count;
  p.n_dyn = a->n_dyn;
  p.k_dyn = a->k_dyn;
  p.b_batched = a->b_batched;
  p.col_index = a->col_index;
  p.col_index_ld = a->col_index_ld;
  p.list_expand = a->row_mode == ROWS_PATCH && a->list_expand > 1 ? a->list_expand : 0;
  p.b_gather = a->b_gather;
  p.b_index = a->b_index;
  p.b_index_ld = a->b_index_ld;
  p.b_rows = a->b_rows;
  if (a->b_gather) {
    if (a->b_gather != B_GATHER_N && a->b_gather != B_GATHER_K) return fail(LAUD_ERR_ARG, "b_gather must be 0, 1 or 2");
    if (!a->b_index || !a->chan_count || a->sample_rows <= 0 || a->b_batched || a->groups > 1 || a->fp32 ||
        a->b_rows <= 0)
      return fail(LAUD_ERR_ARG, "gathered weights need b_index, b_rows, chan_count and sample_rows (no groups / fp32)");
    if (a->b_gather == B_GATHER_K && (a->ksize != 1 || !a->k_dyn || !a->a_compact))
      return fail(LAUD_ERR_ARG, "K-gathered weights: 1x1 conv over compact rows with k_dyn");
    if (a->b_gather == B_GATHER_N && !a->n_dyn) return fail(LAUD_ERR_ARG, "N-gathered weights need n_dyn");
  }
  if (a->sample_rows % 128) return fail(LAUD_ERR_ARG, "sample_rows must be a multiple of 128");
  if ((a->n_dyn || a->k_dyn) && !a->chan_count) return fail(LAUD_ERR_ARG, "chan_count missing");
  p.misplace_first = a->misplace_first;
  p.mdot_w = a->mdot_w;
  p.mdot_out = a->mdot_out;
  p.trace = g_trace;
  static const int dbg_env = [] {
    const char* e = getenv("LAUD_DBG");
    return e ? atoi(e) : 0;
  }();
  p.dbg = dbg_env;
  if (a->fp32) {  // fp32 mode: SIMT FFMA engine, same rows/epilogues (conv_f32.cu)
    if (a->sample_rows || a->chan_count || a->b_batched || a->col_index || a->mdot_w)
      return fail(LAUD_ERR_UNSUPPORTED, "fp32 mode: no per-sample / dynamic-width convs");
    if ((reinterpret_cast<uintptr_t>(a->act) | reinterpret_cast<uintptr_t>(a->weight)) & 15)
      return fail(LAUD_ERR_ARG, "fp32 mode: 16-byte aligned activations and weights");
    p.weight_f32 = a->weight;
    ProfScope ps(0, st, a->row_mode != ROWS_DENSE ? a->count : nullptr);
    return cuda_check(launch_conv_f32(p, st), "conv_f32 launch", 1);
  }
  // Patch conv2 with the halo in shared memory (patch_conv.cu): stride-1 3x3
  // over S = 2 / 4 patches, compact output rows, plain affine epilogue
  static const int halo_env = [] {
    const char* e = getenv("LAUD_HALO");  // bit 0: halo conv2, bit 1: also grouped conv2
    return e ? atoi(e) : 3;
  }();
  if (halo_env && !ad && a->row_mode == ROWS_PATCH && a->ksize == 3 && a->stride == 1 && a->pad == 1 &&
      (p.groups == 1 || (halo_env & 2)) && !a->a_compact && !a->sample_rows && !a->chan_count && !a->b_batched &&
      a->out_mode == OUT_ROW && !a->resid && !a->ymask_coarse && !a->mdot_w &&
      !a->relu_inactive_coarse && !a->out_f32 && !a->col_index && !a->misplace_first &&
      a->patch_h == a->patch_w && a->in_h == a->out_h && a->in_w == a->out_w && a->n_out <= 512 &&
      (reinterpret_cast<uintptr_t>(a->act) % 16) == 0 && (long long)a->batch * a->in_h * a->in_w < (1ll << 31) - 1) {
    const int s = a->patch_h;
    static const int gbn_env = [] {  // N tile of the grouped halo conv (tools: A/B)
      const char* e = getenv("LAUD_PC_GBN");
      return e ? atoi(e) : 128;
    }();
    // grouped: 128-wide N tiles (fewer re-loads of a channel block's halo by the
    // N tiles whose groups straddle it; measured 18.3 -> 17.7 ms on RegNetY b1024)
    static const int pbn_env = [] {  // N tile of the ungrouped S = 2 halo conv (tools: A/B)
      const char* e = getenv("LAUD_PC_BN");
      return e ? atoi(e) : 128;
    }();
    const int hbn = p.groups > 1 ? gbn_env : (s == 4 ? 64 : (a->n_out % 128 == 0 ? pbn_env : 64));
    if (patch_conv_supported(s, hbn)) {
      p.a_rows = a->batch * a->in_h * a->in_w;
      int rc;
      CUtensorMap ma, mb;
      const int kw = 9 * p.kpad;
      if ((rc = tensor_map_2d(a->act, p.a_rows, a->in_c, a->in_ld, 1, &ma)) ||
          (rc = tensor_map_2d(a->weight, a->n_out, kw, kw, hbn, &mb)))
        return rc;
      // split-K over a cluster when one wave of tiles leaves most SMs idle
      const long long pc_tiles = ((long long)(a->rows_max / (s * s)) + 128 / s - 1) / (128 / s) * ((a->n_out + hbn - 1) / hbn);
      const int ncb = p.kpad / 64;
      p.ksplit = 1;
      static const int ks_max = [] {
        const char* e = getenv("LAUD_KSPLIT_MAX");
        return e ? atoi(e) : 8;
      }();
      if (a->latency_split && p.groups == 1)
        for (int k = ks_max; k >= 2; k >>= 1)
          if (ncb % k == 0 && pc_tiles * k <= num_sms()) {
            p.ksplit = k;
            break;
          }
      // larger grids: split only the last partial wave's tiles over 2-CTA clusters
      static const int tail_env = [] {
        const char* e = getenv("LAUD_TAIL_SPLIT");
        return e ? atoi(e) : 1;
      }();
      p.tail_split = (tail_env && a->latency_split && p.groups == 1 && p.ksplit == 1 && ncb % 2 == 0) ? 1 : 0;
      ProfScope ps(0, st, a->count);
      if (ps.on) {
        ps.rec.rows_per_count = (long long)s * s;
        ps.rec.rows_max = a->rows_max;
        ps.rec.n_out = a->n_out;
        ps.rec.k_alg = 9LL * a->in_c / p.groups;  // grouped: C_in / groups per output
        ps.rec.taps = 9;
        ps.rec.resid = 0;
      }
      return cuda_check(launch_patch_conv(ma, mb, p, s, hbn, num_sms(), st), "patch conv launch", 1);
    }
  }
  // grouped: narrow tiles keep the block-diagonal K window short; gathered
  // weights: 128-wide N tiles (the per-sample kept width at r <= 0.5)
  const int bn = p.groups > 1 ? 64
                 : a->b_gather ? (a->n_out <= 64 ? 64 : 128)
                               : pick_bn(a->n_out, a->ksize * a->ksize * round_up(a->in_c, 64), a->rows_max);
  const int kw = a->ksize * a->ksize * p.kpad;
  int rc;
  // A operand: [a_rows][in_c] with row stride in_ld, gathered 4 rows at a time
  CUtensorMap ma;
  memset(&ma, 0, sizeof(ma));
  static const int a_tma_env = [] {
    const char* e = getenv("LAUD_A_TMA");
    return e ? atoi(e) : 1;
  }();
  p.a_tma = a_tma_env && (reinterpret_cast<uintptr_t>(a->act) % 16 == 0);
  if (p.a_tma) {
    const long long arows =
        a->a_compact ? (a->sample_rows > 0 ? (long long)a->batch * a->out_h * a->out_w
                                           : (long long)a->rows_max)
                     : (long long)a->batch * a->in_h * a->in_w;
    if (arows >= (1ll << 31) - 1) {
      p.a_tma = 0;
    } else {
      p.a_rows = (int)arows;
      // contiguous A rows: compact rows, or a dense stride-1 1x1 conv on one grid
      static const int a_tile_env = [] {
        const char* e = getenv("LAUD_A_TILE");
        return e ? atoi(e) : 1;
      }();
      p.a_tile = a_tile_env && a->ksize == 1 &&
                 (a->a_compact || (a->row_mode == ROWS_DENSE && a->sample_rows == 0 &&
                                   a->stride == 1 && a->pad == 0 && a->in_h == a->out_h &&
                                   a->in_w == a->out_w));
      // S x S patches of a 3x3 conv: one 4D box per patch and tap instead of S*S/4 gathers
      static const int a_box_env = [] {
        const char* e = getenv("LAUD_A_BOX");  // bit 0: S = 4, bit 1: S = 2
        return e ? atoi(e) : 1;
      }();
      const int s_box = a->patch_h;
      p.a_box = a->row_mode == ROWS_PATCH && a->ksize == 3 && !a->a_compact && a->patch_h == a->patch_w &&
                ((s_box == 4 && (a_box_env & 1)) || (s_box == 2 && (a_box_env & 2))) &&
                a->in_ld % 8 == 0 && !a->sample_rows && a->stride * s_box <= 256;
      if (p.a_box) {
        if ((rc = tensor_map_patch(a->act, a->batch, a->in_h, a->in_w, a->in_c, a->in_ld, s_box, a->stride, &ma)))
          return rc;
      } else if ((rc = tensor_map_2d(a->act, p.a_rows, a->in_c, a->in_ld, p.a_tile ? 128 : 1, &ma))) {
        return rc;
      }
    }
  }
  // CTA pairs (cta_group::2, M = 256): long-K wide tiles with contiguous A rows and
  // enough rows to fill the TPCs (measured: short K loses, gathered A gains nothing)
  static const int pair_env = [] {
    const char* e = getenv("LAUD_PAIR");  // bit 0: long-K pairs, bit 1: short-K pairs
    return e ? atoi(e) : 1;  // short-K pairs (2) measured slower: opt-in
  }();
  const long long pair_tiles = (long long)((a->rows_max + 255) / 256) * ((a->n_out + bn - 1) / bn);
  const bool pair_ok = pair_env && bn == 256 && p.a_tile && !a->sample_rows && !a->chan_count && !a->b_gather &&
                       !a->b_batched && p.groups == 1 && pair_tiles >= num_sms() / 2;
  const int pair = (!pair_ok || ad) ? 0 : (kw >= 1024 ? 1 : (kw <= 512 && (pair_env & 2) ? 2 : 0));
  // small grids (latency_split): cluster split-K for the plain epilogues — the
  // KS CTAs of a cluster take K slices of one tile, partials reduced over DSMEM
  {
    static const int gks_env = [] {
      const char* e = getenv("LAUD_GEMM_KSPLIT_MAX");
      return e ? atoi(e) : 8;
    }();
    // the split is sized as for a batch of at least 8, so every batch of up to 8
    // images runs the same K slices: the per-row arithmetic (and so the masker
    // decisions downstream) does not depend on how images are batched
    const long long rows_b8 = a->batch > 0 && a->batch < 8 ? (long long)a->rows_max / a->batch * 8 : a->rows_max;
    const long long g_tiles = ((rows_b8 + 127) / 128) * ((a->n_out + bn - 1) / bn);
    const int g_kb = a->ksize * a->ksize * (p.kpad / 64);
    const int npad = (a->n_out + bn - 1) / bn * bn;
    const bool plain = !a->out_f32 && !a->scale && !a->col_index && !a->ymask_coarse && !a->mdot_w &&
                       !a->ymask_channel && !a->relu_inactive_coarse && npad <= 3072;  // VEC_CACHE_FLOATS
    if (gks_env > 1 && bn == 64 && a->latency_split && !pair && !ad && plain && !a->b_gather && !a->chan_count &&
        !a->sample_rows && p.groups == 1)
      for (int k = gks_env >= 8 ? 8 : gks_env >= 4 ? 4 : 2; k >= 2; k >>= 1)
        if (g_tiles * k <= num_sms() && g_kb >= 2 * k) {
          p.ksplit = k;
          break;
        }
  }
  if (ad) {  // fused masker readers need single-CTA tiles with contiguous (TMA box) A rows
    if (!p.a_tile) return LAUD_ADOT_UNAVAILABLE;
    p.adot_w = ad->w;
    p.adot_out = ad->out;
  }
  CUtensorMap m;
  memset(&m, 0, sizeof(m));
  if (a->b_gather) {  // gathered rows are read with cp.async (no tensor map)
    if (a->b_gather == B_GATHER_K && a->n_out % 64)
      return fail(LAUD_ERR_SHAPE, "K-gathered weights: n_out must be a multiple of 64");
    if (reinterpret_cast<uintptr_t>(a->weight) % 16) return fail(LAUD_ERR_ARG, "gathered weights: 16-byte alignment");
    p.weight_g = a->weight;
    p.b_ld = a->b_gather == B_GATHER_N ? kw : a->n_out;
  } else if ((rc = tensor_map_2d(a->weight, a->n_out, kw, kw, pair ? bn / 2 : bn, &m, a->b_batched ? a->batch : 0))) {
    return rc;
  }
  // TMA-store epilogue (plain epilogues only; the kernel ignores it otherwise):
  // dense rows as 32-row boxes, scattered S x S patches (S >= 2) as pixel boxes
  CUtensorMap mo;
  memset(&mo, 0, sizeof(mo));
  static const int tma_out_env = [] {
    const char* e = getenv("LAUD_TMA_OUT");
    return e ? atoi(e) : 1;
  }();
  const bool out_ok = tma_out_env && !a->out_f32 && !a->col_index && (reinterpret_cast<uintptr_t>(a->out) & 15) == 0;
  if (out_ok && a->row_mode == ROWS_DENSE && a->out_mode == OUT_ROW && !a->sample_rows && !a->count) {
    if (tensor_map_2d(a->out, a->rows_max, a->n_out, a->out_ld, 32, &mo) == LAUD_OK) p.tma_out = 1;
  } else if (out_ok && a->row_mode == ROWS_PATCH && a->out_mode == OUT_PIXEL && a->patch_h == a->patch_w &&
             a->patch_h >= 2 && a->patch_h <= 4) {
    if (tensor_map_patch(a->out, a->batch, a->out_h, a->out_w, a->n_out, a->out_ld, a->patch_h, 1, &mo) == LAUD_OK)
      p.tma_out = 2;
  }
  ProfScope ps(0, st, a->row_mode != ROWS_DENSE ? a->count : nullptr);
  if (ps.on) {
    ps.rec.rows_per_count = a->row_mode == ROWS_PATCH ? (long long)p.patch_h * p.patch_w : 1;
    ps.rec.rows_max = a->rows_max;
    ps.rec.n_out = a->n_out;
    ps.rec.k_alg = (long long)a->ksize * a->ksize * a->in_c / p.groups;  // grouped: C_in / groups per output
    ps.rec.taps = a->ksize * a->ksize;
    ps.rec.resid = a->resid != nullptr;
  }
  return cuda_check(launch_conv_gemm(ma, m, mo, bn, p, num_sms(), st, pair), "conv_gemm launch", 1);
}

}  // namespace

extern "C" {

void laud_profile_begin(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (!g_prof_counts) cudaMalloc(&g_prof_counts, kProfSnaps * sizeof(int));
  g_prof_nsnap = 0;
  g_prof_on = true;
}

int laud_profile_end(laud_profile_record* out, int max_records) {
  std::vector<ProfRec> recs;
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_on = false;
    recs.swap(g_prof);
  }
  int n = 0;
  std::vector<int> snaps(kProfSnaps, 0);
  cudaDeviceSynchronize();
  if (g_prof_counts && g_prof_nsnap)
    cudaMemcpy(snaps.data(), g_prof_counts, g_prof_nsnap * sizeof(int), cudaMemcpyDeviceToHost);
  for (auto& r : recs) {
    cudaEventSynchronize(r.e1);
    if (out && n < max_records) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, r.e0, r.e1);
      long long rows = r.rows_max;
      if (r.snap >= 0) {
        rows = (long long)snaps[r.snap] * r.rows_per_count;
        if (rows > r.rows_max) rows = r.rows_max;
      }
      out[n].tag = r.tag;
      out[n].ms = ms;
      out[n].rows = rows;
      out[n].n_out = r.n_out;
      out[n].k = r.k_alg;
      out[n].bytes = r.bytes;
      out[n].taps = r.taps;
      out[n].resid = r.resid;
      ++n;
    }
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  return n;
}

void laud_debug_set_trace(void* dev_buf) { g_trace = static_cast<unsigned long long*>(dev_buf); }

const char* laud_version(void) { return "laud-b200 0.1.0 (sm_100a, tcgen05)"; }
const char* laud_last_error(void) { return g_err.c_str(); }
uint64_t laud_launch_count(void) { return g_launches.load(); }

size_t laud_scan_workspace_bytes(int items) { return scan_state_bytes(items > 0 ? items : 1); }

size_t laud_masker_partial_floats(int n, int h, int w, int c, int s, int stride) {
  const int win = s * stride;
  if (win <= 0 || h % win || w % win) return 0;
  int cps = 0;
  const int splits = masker_splits(win, c, &cps);
  return (size_t)n * (h / win) * (w / win) * splits;
}

int laud_spatial_masker(const void* x, int x_f32, int ld, int n, int h, int w, int c, int s,
                        int stride, const float* wdiff, float bias, uint8_t* coarse,
                        int* cell_list, int* cell_count, float* partial, void* scan,
                        void* stream) {
  if (s < 1 || stride < 1) return fail(LAUD_ERR_ARG, "granularity and stride must be positive");
  const int win = s * stride;
  if (h % win || w % win)
    return fail(LAUD_ERR_GRANULARITY, "S=%d (window %d) does not divide %dx%d", s, win, h, w);
  if (c % 8 || ld % 8 || ld < c) return fail(LAUD_ERR_SHAPE, "channels must be multiples of 8");
  if (c > 12288) return fail(LAUD_ERR_SHAPE, "masker supports at most 12288 channels");
  ProfScope ps(1, (cudaStream_t)stream);
  if (ps.on) ps.rec.bytes = (long long)n * h * w * c * (x_f32 ? 4 : 2);
  return cuda_check(launch_spatial_masker(x, x_f32, ld, n, h, w, c, s, stride, wdiff, bias, coarse,
                                          cell_list, cell_count, partial, scan,
                                          (cudaStream_t)stream, nullptr, nullptr),
                    "spatial masker", 2);
}

int laud_cells_from_mask(const uint8_t* coarse, int cells, int* cell_list, int* cell_count,
                         void* scan, void* stream) {
  ProfScope ps(2, (cudaStream_t)stream);
  if (ps.on) ps.rec.bytes = (long long)cells * 5;
  return cuda_check(
      launch_list_from_mask(coarse, cells, cell_list, cell_count, scan, (cudaStream_t)stream),
      "cells from mask", 1);
}

int laud_dilate_pixels(const uint8_t* coarse, int n, int h_in, int w_in, int s, int stride,
                       int radius, int* pix_list, int* pix_count, void* scan, void* stream) {
  const int win = s * stride;
  if (s < 1 || stride < 1 || h_in % win || w_in % win)
    return fail(LAUD_ERR_GRANULARITY, "S=%d does not divide the output grid", s);
  if (radius < 0) return fail(LAUD_ERR_ARG, "radius must be >= 0");
  ProfScope ps(2, (cudaStream_t)stream);
  if (ps.on) ps.rec.bytes = (long long)n * h_in * w_in * 4;
  return cuda_check(launch_dilate_pixels(coarse, n, h_in, w_in, s, stride, h_in / win, w_in / win,
                                         radius, pix_list, pix_count, scan, (cudaStream_t)stream),
                    "dilate pixels", 1);
}

int laud_conv(const laud_conv_args* a, void* stream) { return run_conv(a, (cudaStream_t)stream); }

static int round64(int v) { return (v + 63) / 64 * 64; }

int laud_channel_masker(const void* x, int x_f32, int ld, int n, int hw, int c, const float* w1,
                        int hidden, const float* w2, int d, int g, int cm, int cm_p,
                        uint8_t* coarse, float* dvals, uint8_t* expanded, int* sel, int* count,
                        const float* bias, void* stream) {
  if (c % 8 || ld % 8 || ld < c) return fail(LAUD_ERR_SHAPE, "channels must be multiples of 8");
  if (d < 1 || g < 1 || cm != d * g || cm > cm_p) return fail(LAUD_ERR_GRANULARITY, "bad D/G");
  if ((size_t)(c + hidden + d + 8 * 1024) * 4 > 100 * 1024) return fail(LAUD_ERR_SHAPE, "masker too wide");
  ProfScope ps(1, (cudaStream_t)stream);
  return cuda_check(launch_channel_masker(x, x_f32, ld, n, hw, c, w1, hidden, w2, d, g, cm, cm_p,
                                          coarse, dvals, expanded, sel, count, bias,
                                          (cudaStream_t)stream),
                    "channel masker", 1);
}

size_t laud_channel_pack_bytes(int n, int c_in, int c_mid, int c_out) {
  const size_t w1 = (size_t)c_mid * round64(c_in);
  const size_t w2 = (size_t)c_mid * 9 * round64(c_mid);
  const size_t w3 = (size_t)c_out * round64(c_mid);
  return (size_t)n * (w1 + w2 + w3) * 2 + 256;
}

// Channel skipping (`reference.py:404-423`): per sample, conv1 over the kept
// filters W1[sel], conv2 with W2[sel][:, sel], conv3 with W3[:, sel] — packed
// per sample, run as dynamic-width tcgen05 GEMMs (ragged N / K per sample).
static int channel_forward(const laud_block_args* a, cudaStream_t st) {
  const int n = a->n, cmp = a->c_mid;
  const int ho = (a->h_in - 1) / a->stride + 1, wo = (a->w_in - 1) / a->stride + 1;
  if (!a->ch_sel || !a->ch_count || !a->ch_expanded || !a->wpack || !a->h1 || !a->h2)
    return fail(LAUD_ERR_ARG, "channel workspace missing");
  int rc;
  if (a->given_chmask) {
    if ((rc = cuda_check(launch_channel_lists(a->given_chmask, n, cmp, a->ch_sel, a->ch_count, st),
                         "channel lists", 1)))
      return rc;
  } else {
    if (!a->ch_w1 || !a->ch_w2 || !a->ch_coarse || a->ch_d < 1 || a->ch_groups < 1)
      return fail(LAUD_ERR_ARG, "channel masker weights missing");
    const int cm = a->ch_d * a->ch_groups;
    if (cm > cmp) return fail(LAUD_ERR_GRANULARITY, "D*G exceeds the mid width");
    ProfScope ps(1, st);
    if ((rc = cuda_check(launch_channel_masker(a->x, a->fp32, a->x_ld, n, a->h_in * a->w_in, a->c_in,
                                               a->ch_w1, a->ch_hidden, a->ch_w2, a->ch_d,
                                               a->ch_groups, cm, cmp, a->ch_coarse, a->ch_dvals,
                                               a->ch_expanded, a->ch_sel, a->ch_count, a->ch_bias,
                                               st),
                         "channel masker", 1)))
      return rc;
  }
  // skip path
  if (a->has_down) {
    laud_conv_args d;
    memset(&d, 0, sizeof(d));
    d.fp32 = a->fp32;
    d.row_mode = ROWS_DENSE;
    d.rows_max = n * ho * wo;
    d.batch = n;
    d.out_h = ho;
    d.out_w = wo;
    d.act = a->x;
    d.in_h = a->h_in;
    d.in_w = a->w_in;
    d.in_c = a->c_in;
    d.in_ld = a->x_ld;
    d.ksize = 1;
    d.stride = a->stride;
    d.weight = a->wd;
    d.n_out = a->c_out;
    d.scale = a->sd;
    d.bias = a->bd;
    d.out_mode = OUT_PIXEL;
    d.out = a->out;
    d.out_ld = a->c_out;
    if ((rc = run_conv(&d, st))) return rc;
  } else if (a->out != a->x) {
    if ((rc = cuda_check(cudaMemcpyAsync(a->out, a->x, (size_t)n * ho * wo * a->c_out * (a->fp32 ? 4 : 2),
                                         cudaMemcpyDeviceToDevice, st),
                         "skip copy", 0)))
      return rc;
  }
  static const int dense_min = [] {
    const char* e = getenv("LAUD_CH_DENSE_MIN");
    return e ? atoi(e) : 8;
  }();
  // EXT schedule (opt-in, LAUD_CH_GATHER=1): per-sample weights gathered
  // inside the conv kernels instead of a packing pass.  conv1 stays
  // dense-masked (h1 full width, zero on the dropped channels); conv2's tiles
  // belong to one sample and gather their B rows W2[sel] (N = k_n, K = the
  // full masked h1 -> r F2); h2 is compact (k_n columns, sel order); conv3
  // gathers the K rows of W3^T (MN-major B: K = k_n -> r F3) and adds into
  // the residual.  Correct (tests) but measured slower than the dense-masked
  // schedule at batch 256 (R101 stage-3 conv2: 381 us gathered vs 83 us
  // dense, tools/engine_probe.py chconv2_s3): the per-(tile, k-block) weight
  // gather (16 KiB from scattered rows, TMA gather4 or cp.async) is far below
  // the MMA rate, and a sample's 196 rows cannot amortise it.
  // Read per call so tests can switch it.
  const char* ge = getenv("LAUD_CH_GATHER");
  const int gather_env = ge ? atoi(ge) : 0;
  const int hw2 = ho * wo, sr2g = (hw2 + 127) / 128 * 128;
  if (gather_env && !a->fp32 && a->groups == 1 && a->w3t && dense_min > 0 && n >= dense_min &&
      sr2g * 100 <= hw2 * 135 && a->c_out % 64 == 0) {
    laud_conv_args c1;
    memset(&c1, 0, sizeof(c1));
    c1.row_mode = ROWS_DENSE;
    c1.rows_max = n * a->h_in * a->w_in;
    c1.batch = n;
    c1.out_h = a->h_in;
    c1.out_w = a->w_in;
    c1.patch_h = c1.patch_w = c1.cells_h = c1.cells_w = 1;
    c1.act = a->x;
    c1.in_h = a->h_in;
    c1.in_w = a->w_in;
    c1.in_c = a->c_in;
    c1.in_ld = a->x_ld;
    c1.ksize = 1;
    c1.stride = 1;
    c1.weight = a->w1;
    c1.n_out = cmp;
    c1.scale = a->s1;
    c1.bias = a->b1;
    c1.relu = a->relu1;
    c1.ymask_channel = a->ch_expanded;
    c1.out_mode = OUT_PIXEL;
    c1.out = a->h1;
    c1.out_ld = cmp;
    if ((rc = run_conv(&c1, st))) return rc;
    laud_conv_args c2;
    memset(&c2, 0, sizeof(c2));
    c2.row_mode = ROWS_DENSE;
    c2.sample_rows = sr2g;
    c2.rows_max = n * sr2g;
    c2.batch = n;
    c2.out_h = ho;
    c2.out_w = wo;
    c2.patch_h = c2.patch_w = c2.cells_h = c2.cells_w = 1;
    c2.act = a->h1;
    c2.in_h = a->h_in;
    c2.in_w = a->w_in;
    c2.in_c = cmp;
    c2.in_ld = cmp;
    c2.ksize = 3;
    c2.stride = a->stride;
    c2.pad = 1;
    c2.weight = a->w2;
    c2.n_out = cmp;
    c2.chan_count = a->ch_count;
    c2.n_dyn = 1;
    c2.col_index = a->ch_sel;
    c2.col_index_ld = cmp;
    c2.b_gather = B_GATHER_N;
    c2.b_index = a->ch_sel;
    c2.b_index_ld = cmp;
    c2.b_rows = cmp;
    c2.scale = a->s2;
    c2.bias = a->b2;
    c2.relu = a->relu2;
    c2.out_mode = OUT_ROW;
    c2.out = a->h2;
    c2.out_ld = cmp;
    if ((rc = run_conv(&c2, st))) return rc;
    if (a->se_w1) {  // EXT squeeze-excitation over each sample's kept channels (compact h2)
      if ((rc = cuda_check(launch_se_channel(a->h2, n, cmp, hw2, hw2, a->ch_sel, a->ch_count, a->se_w1,
                                             a->se_b1, a->se_hidden, a->se_w2, a->se_b2, a->h1, st),
                           "squeeze-excitation (channel)", 1)))
        return rc;
    }
    laud_conv_args c3;
    memset(&c3, 0, sizeof(c3));
    c3.row_mode = ROWS_DENSE;
    c3.sample_rows = sr2g;
    c3.rows_max = n * sr2g;
    c3.batch = n;
    c3.out_h = ho;
    c3.out_w = wo;
    c3.patch_h = c3.patch_w = c3.cells_h = c3.cells_w = 1;
    c3.act = a->h2;
    c3.in_h = ho;
    c3.in_w = wo;
    c3.in_c = cmp;
    c3.in_ld = cmp;
    c3.a_compact = 1;
    c3.ksize = 1;
    c3.stride = 1;
    c3.weight = a->w3t;
    c3.n_out = a->c_out;
    c3.chan_count = a->ch_count;
    c3.k_dyn = 1;
    c3.b_gather = B_GATHER_K;
    c3.b_index = a->ch_sel;
    c3.b_index_ld = cmp;
    c3.b_rows = cmp;
    c3.scale = a->s3;
    c3.bias = a->b3;
    c3.relu = a->relu_out;
    c3.out_mode = OUT_PIXEL;
    c3.out = a->out;
    c3.out_ld = a->c_out;
    c3.resid = a->out;
    c3.resid_ld = a->c_out;
    return run_conv(&c3, st);
  }
  // Schedule.  Per-sample dynamic width (below) computes exactly the kept
  // channels but packs W1[sel], W2[sel][:, sel], W3[:, sel] for every sample —
  // at large batch that weight traffic (n * r|W|) dwarfs the activations, so
  // from LAUD_CH_DENSE_MIN samples on (and in fp32 mode) the block runs the
  // dense-masked schedule of the same algebra (reference.py:336-339): dense
  // convs, h1 and h2 zeroed on the dropped channels in the epilogues, so conv3
  // sums only the kept ones.
  if (a->fp32 || (dense_min > 0 && n >= dense_min)) {
    laud_conv_args c1;
    memset(&c1, 0, sizeof(c1));
    c1.fp32 = a->fp32;
    c1.row_mode = ROWS_DENSE;
    c1.rows_max = n * a->h_in * a->w_in;
    c1.batch = n;
    c1.out_h = a->h_in;
    c1.out_w = a->w_in;
    c1.patch_h = c1.patch_w = c1.cells_h = c1.cells_w = 1;
    c1.act = a->x;
    c1.in_h = a->h_in;
    c1.in_w = a->w_in;
    c1.in_c = a->c_in;
    c1.in_ld = a->x_ld;
    c1.ksize = 1;
    c1.stride = 1;
    c1.weight = a->w1;
    c1.n_out = cmp;
    c1.scale = a->s1;
    c1.bias = a->b1;
    c1.relu = a->relu1;
    c1.ymask_channel = a->ch_expanded;
    c1.out_mode = OUT_PIXEL;
    c1.out = a->h1;
    c1.out_ld = cmp;
    if ((rc = run_conv(&c1, st))) return rc;
    laud_conv_args c2 = c1;
    c2.rows_max = n * ho * wo;
    c2.out_h = ho;
    c2.out_w = wo;
    c2.act = a->h1;
    c2.in_c = cmp;
    c2.in_ld = cmp;
    c2.ksize = 3;
    c2.stride = a->stride;
    c2.pad = 1;
    c2.weight = a->w2;  // the grouped kernel itself: masking is multiplicative
    c2.groups = a->groups;
    c2.scale = a->s2;
    c2.bias = a->b2;
    c2.relu = a->relu2;
    c2.out_mode = OUT_ROW;
    c2.out = a->h2;
    // conv2 (stride 1) on the halo kernel over an identity cell list, the channel
    // mask in its epilogue; conv3 reads h2 in the same patch order
    if (!a->fp32 && a->stride == 1) {
      const int sc = cmp <= 64 ? 4 : 2;
      if (ho % sc == 0 && wo % sc == 0 && cmp <= 512) {
        const int* iota = identity_list(n * (ho / sc) * (wo / sc), st);
        if (iota) {
          c2.row_mode = ROWS_PATCH;
          c2.list = iota;
          c2.count = nullptr;
          c2.patch_h = c2.patch_w = sc;
          c2.cells_h = ho / sc;
          c2.cells_w = wo / sc;
        }
      }
    }
    if ((rc = run_conv(&c2, st))) return rc;
    if (a->se_w1) {  // EXT SE on the dense-masked h2 (dropped channels pool to zero)
      if ((rc = cuda_check(launch_se(a->h2, n, cmp, nullptr, nullptr, 1, 1, ho * wo, a->se_w1, a->se_b1,
                                     a->se_hidden, a->se_w2, a->se_b2, a->h1, st),
                           "squeeze-excitation (channel)", 1)))
        return rc;
    }
    laud_conv_args c3 = c2;
    c3.groups = 1;
    c3.act = a->h2;
    c3.in_h = ho;
    c3.in_w = wo;
    c3.a_compact = 1;
    c3.ksize = 1;
    c3.stride = 1;
    c3.pad = 0;
    c3.weight = a->w3;
    c3.n_out = a->c_out;
    c3.ymask_channel = nullptr;
    c3.scale = a->s3;
    c3.bias = a->b3;
    c3.relu = a->relu_out;
    c3.out_mode = OUT_PIXEL;
    c3.out = a->out;
    c3.out_ld = a->c_out;
    c3.resid = a->out;
    c3.resid_ld = a->c_out;
    return run_conv(&c3, st);
  }
  // per-sample packed weights
  const int k1 = round64(a->c_in), k2 = round64(cmp);
  char* wp = reinterpret_cast<char*>(a->wpack);
  void* w1s = wp;
  void* w2s = wp + (size_t)n * cmp * k1 * 2;
  void* w3s = wp + (size_t)n * cmp * k1 * 2 + (size_t)n * cmp * 9 * k2 * 2;
  {
    ProfScope ps(3, st);
    if ((rc = cuda_check(launch_pack_weights(a->w1, cmp, 1, k1, w1s, cmp, k1, a->ch_sel, a->ch_count,
                                             cmp, 1, 0, n, st), "pack w1", 1)) ||
        (rc = cuda_check(launch_pack_weights(a->groups > 1 ? a->w2_dense : a->w2, cmp, 9, k2, w2s, cmp, k2, a->ch_sel, a->ch_count,
                                             cmp, 1, 1, n, st), "pack w2", 1)) ||
        (rc = cuda_check(launch_pack_weights(a->w3, a->c_out, 1, k2, w3s, a->c_out, k2, a->ch_sel,
                                             a->ch_count, cmp, 0, 1, n, st), "pack w3", 1)))
      return rc;
  }
  const int sr1 = (a->h_in * a->w_in + 127) / 128 * 128;
  const int sr2 = (ho * wo + 127) / 128 * 128;
  laud_conv_args c1;
  memset(&c1, 0, sizeof(c1));
  c1.fp32 = a->fp32;
  c1.row_mode = ROWS_DENSE;
  c1.sample_rows = sr1;
  c1.rows_max = n * sr1;
  c1.batch = n;
  c1.out_h = a->h_in;
  c1.out_w = a->w_in;
  c1.act = a->x;
  c1.in_h = a->h_in;
  c1.in_w = a->w_in;
  c1.in_c = a->c_in;
  c1.in_ld = a->x_ld;
  c1.ksize = 1;
  c1.stride = 1;
  c1.weight = w1s;
  c1.b_batched = 1;
  c1.n_out = cmp;
  c1.chan_count = a->ch_count;
  c1.n_dyn = 1;
  c1.col_index = a->ch_sel;
  c1.col_index_ld = cmp;
  c1.scale = a->s1;
  c1.bias = a->b1;
  c1.relu = a->relu1;
  c1.out_mode = OUT_ROW;
  c1.out = a->h1;
  c1.out_ld = cmp;
  if ((rc = run_conv(&c1, st))) return rc;
  laud_conv_args c2 = c1;
  c2.sample_rows = sr2;
  c2.rows_max = n * sr2;
  c2.out_h = ho;
  c2.out_w = wo;
  c2.act = a->h1;
  c2.in_c = cmp;
  c2.in_ld = cmp;
  c2.ksize = 3;
  c2.stride = a->stride;
  c2.pad = 1;
  c2.weight = w2s;
  c2.k_dyn = 1;
  c2.scale = a->s2;
  c2.bias = a->b2;
  c2.relu = a->relu2;
  c2.out = a->h2;
  if ((rc = run_conv(&c2, st))) return rc;
  if (a->se_w1) {  // EXT squeeze-excitation over each sample's kept channels
    // (conv2 wrote sample n's rows compactly at [n*ho*wo, (n+1)*ho*wo))
    if (a->c_mid % 8 || (size_t)n * sr1 * cmp * 2 < (size_t)2 * n * cmp * 4)
      return fail(LAUD_ERR_SHAPE, "SE needs c_mid % 8 == 0");
    if ((rc = cuda_check(launch_se_channel(a->h2, n, cmp, ho * wo, ho * wo, a->ch_sel, a->ch_count, a->se_w1,
                                           a->se_b1, a->se_hidden, a->se_w2, a->se_b2, a->h1, st),
                         "squeeze-excitation (channel)", 1)))
      return rc;
  }
  laud_conv_args c3 = c2;
  c3.act = a->h2;
  c3.in_h = ho;
  c3.in_w = wo;
  c3.a_compact = 1;
  c3.ksize = 1;
  c3.stride = 1;
  c3.pad = 0;
  c3.weight = w3s;
  c3.n_out = a->c_out;
  c3.n_dyn = 0;
  c3.col_index = nullptr;
  c3.scale = a->s3;
  c3.bias = a->b3;
  c3.relu = a->relu_out;
  c3.out_mode = OUT_PIXEL;
  c3.out = a->out;
  c3.out_ld = a->c_out;
  c3.resid = a->out;
  c3.resid_ld = a->c_out;
  return run_conv(&c3, st);
}

int laud_block_forward(const laud_block_args* a, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!a || !a->x || !a->out || !a->w1 || !a->w2 || !a->w3)
    return fail(LAUD_ERR_ARG, "null pointer in block args");
  if (a->groups < 1) return fail(LAUD_ERR_ARG, "groups must be >= 1");
  if (a->groups != 1 && a->paradigm == LAUD_PARADIGM_CHANNEL && !a->w2_dense)  // reference.py:405-406
    return fail(LAUD_ERR_UNSUPPORTED, "sparse channel execution requires groups == 1");
  if (a->se_w1 && a->paradigm == LAUD_PARADIGM_CHANNEL && a->fp32)
    return fail(LAUD_ERR_UNSUPPORTED, "squeeze-excitation under channel skipping needs bf16 mode");
  if (a->stride != 1 && a->stride != 2) return fail(LAUD_ERR_ARG, "stride must be 1 or 2");
  if (a->stride > 1 && !a->has_down)
    return fail(LAUD_ERR_SHAPE, "a strided block needs a downsample path");
  if (a->has_down && !a->wd) return fail(LAUD_ERR_ARG, "downsample weights missing");
  const int ho = (a->h_in - 1) / a->stride + 1, wo = (a->w_in - 1) / a->stride + 1;
  if (!a->has_down && (a->c_in != a->c_out || a->x_ld != a->c_out))
    return fail(LAUD_ERR_SHAPE, "identity skip needs c_in == c_out == x_ld");
  if (a->paradigm == LAUD_PARADIGM_CHANNEL) return channel_forward(a, st);
  const int n = a->n;
  int rc;
  // masker fused into a dense conv1: its A stages feed the window dots, so x is
  // read once for both (the masker's own pass over x disappears)
  static const int fuse_env = [] {
    const char* e = getenv("LAUD_MASKER_IN_CONV1");
    return e ? atoi(e) : 1;
  }();
  // small grids (latency-bound, e.g. batch 1): the one-launch standalone
  // masker on the auxiliary stream, concurrent with a plain conv1 — its
  // decisions cost no time on the block's critical path (conv1's fused
  // readers would lengthen conv1's single-CTA K loop instead)
  static const int fork_env = [] {
    const char* e = getenv("LAUD_MASKER_FORK");
    return e ? atoi(e) : 1;
  }();
  const bool masker_computed = (a->paradigm == LAUD_PARADIGM_SPATIAL || a->paradigm == LAUD_PARADIGM_LAYER) &&
                               !a->given_coarse && !a->dn && a->masker_wdiff;
  const long long mask_cells =
      a->paradigm == LAUD_PARADIGM_LAYER ? n : (a->s > 0 ? (long long)n * (ho / a->s) * (wo / a->s) : 0);
  const bool fork_masker = fork_env && a->aux_stream && masker_computed && mask_cells <= 4096;
  const bool fuse_masker = fuse_env && !fork_masker && a->paradigm == LAUD_PARADIGM_SPATIAL && a->conv1_dense &&
                           !a->given_coarse && !a->dn && !a->fp32 && a->masker_wdiff && a->cell_sums &&
                           a->x_ld == a->c_in;  // K tail past c_in: zero-filled A, zero weights
  cudaEvent_t fork_done = nullptr;

  // ---------------------------------------------------------------- rows
  int pm;  // row mode for conv2/conv3
  int ph = 1, pw = 1, ch = 1, cw = 1;
  const int* cells = nullptr;
  const int* cells_n = nullptr;
  const uint8_t* coarse = nullptr;
  if (a->paradigm == LAUD_PARADIGM_SPATIAL || a->paradigm == LAUD_PARADIGM_LAYER) {
    if (a->paradigm == LAUD_PARADIGM_SPATIAL) {
      if (a->s < 1 || ho % a->s || wo % a->s)
        return fail(LAUD_ERR_GRANULARITY, "S=%d does not divide %dx%d", a->s, ho, wo);
      ph = pw = a->s;
    } else {
      ph = ho;
      pw = wo;
    }
    ch = ho / ph;
    cw = wo / pw;
    if (!a->cell_list || !a->cell_count || !a->scan)
      return fail(LAUD_ERR_ARG, "cell list / scan workspace missing");
    if (a->given_coarse) {
      coarse = a->given_coarse;
      rc = laud_cells_from_mask(coarse, n * ch * cw, a->cell_list, a->cell_count, a->scan, stream);
    } else if (fuse_masker) {
      // decisions come from conv1's fused dots (below, before the skip path)
      if (!a->coarse_out) return fail(LAUD_ERR_ARG, "coarse output missing");
      coarse = a->coarse_out;
      rc = LAUD_OK;
    } else {
      if (!a->masker_wdiff || !a->coarse_out || !a->partial)
        return fail(LAUD_ERR_ARG, "masker weights / coarse output / partials missing");
      if (a->paradigm == LAUD_PARADIGM_LAYER && a->h_in != a->w_in)
        return fail(LAUD_ERR_GRANULARITY, "layer masker needs a square feature");
      coarse = a->coarse_out;
      if (a->dn) {  // masker-conv3 fusion with the previous block (same grid and S)
        ProfScope ps(1, st);
        rc = cuda_check(launch_spatial_masker(a->x, a->fp32, a->x_ld, n, a->h_in, a->w_in, a->c_in,
                                              a->paradigm == LAUD_PARADIGM_LAYER ? ho : a->s,
                                              a->stride, a->masker_wdiff, a->masker_bias,
                                              a->coarse_out, a->cell_list, a->cell_count,
                                              a->partial, a->scan, st, a->prev_coarse, a->dn),
                        "spatial masker (fused)", 2);
      } else if (fork_masker) {
        cudaStream_t aux = (cudaStream_t)a->aux_stream;
        cudaEvent_t x_ready = fork_event(0);
        fork_done = fork_event(1);
        if ((rc = cuda_check(cudaEventRecord(x_ready, st), "fork record", 0)) ||
            (rc = cuda_check(cudaStreamWaitEvent(aux, x_ready, 0), "fork wait", 0)))
          return rc;
        // the masker kernel itself is launched after conv1 (below): conv1's few
        // CTAs need nearly a whole SM of shared memory each and must not wait
        // behind the masker's small CTAs already resident on every SM
      } else {
        rc = laud_spatial_masker(a->x, a->fp32, a->x_ld, n, a->h_in, a->w_in, a->c_in,
                                 a->paradigm == LAUD_PARADIGM_LAYER ? ho : a->s, a->stride,
                                 a->masker_wdiff, a->masker_bias, a->coarse_out, a->cell_list,
                                 a->cell_count, a->partial, a->scan, stream);
      }
    }
    if (rc) return rc;
    cells = a->cell_list;
    cells_n = a->cell_count;
    pm = ROWS_PATCH;
  } else if (a->paradigm == LAUD_PARADIGM_STATIC) {
    pm = ROWS_DENSE;
  } else {
    return fail(LAUD_ERR_ARG, "unknown paradigm %d", a->paradigm);
  }
  // Static blocks run conv2 on the halo kernel too (every S x S cell active:
  // an identity cell list), measured faster than the gathered-row dense conv2
  // at every R101 stage (tools/engine_probe.py conv2_s* vs pconv_s*_all); the
  // K order is the same, so the outputs are bitwise those of the dense path.
  int pm2 = pm;  // row mode of conv2 / conv3
  {
    static const int sh_env = [] {
      const char* e = getenv("LAUD_STATIC_HALO");
      return e ? atoi(e) : 1;
    }();
    const int sh = a->c_mid <= 64 ? 4 : 2;
    if (sh_env && pm == ROWS_DENSE && !a->fp32 && a->stride == 1 && ho % sh == 0 && wo % sh == 0 &&
        a->c_mid <= 512 && a->c_mid % 8 == 0) {
      const int* iota = identity_list(n * (ho / sh) * (wo / sh), st);
      if (iota) {
        pm2 = ROWS_PATCH;
        ph = pw = sh;
        ch = ho / sh;
        cw = wo / sh;
        cells = iota;
        cells_n = nullptr;
      }
    }
  }

  // ---------------------------------------------------------------- conv1
  laud_conv_args c1;
  memset(&c1, 0, sizeof(c1));
  c1.fp32 = a->fp32;
  c1.batch = n;
  c1.out_h = a->h_in;
  c1.out_w = a->w_in;
  c1.act = a->x;
  c1.in_h = a->h_in;
  c1.in_w = a->w_in;
  c1.in_c = a->c_in;
  c1.in_ld = a->x_ld;
  c1.ksize = 1;
  c1.stride = 1;
  c1.weight = a->w1;
  c1.n_out = a->c_mid;
  c1.scale = a->s1;
  c1.bias = a->b1;
  c1.relu = a->relu1;
  c1.out_mode = OUT_PIXEL;
  c1.out = a->h1;
  c1.out_ld = a->c_mid;
  c1.rows_max = n * a->h_in * a->w_in;
  c1.latency_split = a->latency_split;
  bool conv1_done = false;
  if (fuse_masker) {
    // per-pixel masker dots stored by conv1's readers, then decisions + the
    // active-cell list (reference.py:173-183, 133-135)
    const int win = a->s * a->stride;
    c1.row_mode = ROWS_DENSE;
    AdotArgs ad{a->masker_wdiff, a->cell_sums};
    rc = run_conv(&c1, st, &ad);
    if (rc == LAUD_OK) {
      conv1_done = true;
      ProfScope ps(1, st);
      if ((rc = cuda_check(launch_masker_decide(a->cell_sums, n, a->h_in, a->w_in, win, a->masker_bias,
                                                a->coarse_out, a->cell_list, a->cell_count, a->scan, st),
                           "masker decide", 1)))
        return rc;
    } else if (rc == LAUD_ADOT_UNAVAILABLE) {  // this geometry cannot host it: standalone masker
      if ((rc = laud_spatial_masker(a->x, a->fp32, a->x_ld, n, a->h_in, a->w_in, a->c_in, a->s, a->stride,
                                    a->masker_wdiff, a->masker_bias, a->coarse_out, a->cell_list,
                                    a->cell_count, a->partial, a->scan, stream)))
        return rc;
    } else {
      return rc;
    }
  }

  if (fork_done) {
    // conv1 runs densely on the block's stream while the forked masker
    // decides (for a layer block, inactive samples' h1 is computed but never
    // read); the decisions are joined before the skip path (ReLU at inactive
    // cells) and conv2
    c1.row_mode = ROWS_DENSE;
    if ((rc = run_conv(&c1, st))) return rc;
    conv1_done = true;
    cudaStream_t aux = (cudaStream_t)a->aux_stream;
    if ((rc = laud_spatial_masker(a->x, a->fp32, a->x_ld, n, a->h_in, a->w_in, a->c_in,
                                  a->paradigm == LAUD_PARADIGM_LAYER ? ho : a->s, a->stride, a->masker_wdiff,
                                  a->masker_bias, a->coarse_out, a->cell_list, a->cell_count, a->partial,
                                  a->scan, aux)) ||
        (rc = cuda_check(cudaEventRecord(fork_done, aux), "join record", 0)))
      return rc;
    if ((rc = cuda_check(cudaStreamWaitEvent(st, fork_done, 0), "join wait", 0))) return rc;
  }

  // ---------------------------------------------------------------- skip path
  if (a->has_down) {
    laud_conv_args d;
    memset(&d, 0, sizeof(d));
    d.fp32 = a->fp32;
    d.row_mode = ROWS_DENSE;
    d.rows_max = n * ho * wo;
    d.batch = n;
    d.out_h = ho;
    d.out_w = wo;
    d.patch_h = ph;
    d.patch_w = pw;
    d.cells_h = ch;
    d.cells_w = cw;
    d.act = a->x;
    d.in_h = a->h_in;
    d.in_w = a->w_in;
    d.in_c = a->c_in;
    d.in_ld = a->x_ld;
    d.ksize = 1;
    d.stride = a->stride;
    d.pad = 0;
    d.weight = a->wd;
    d.n_out = a->c_out;
    d.scale = a->sd;
    d.bias = a->bd;
    d.out_mode = OUT_PIXEL;
    d.out = a->out;
    d.out_ld = a->c_out;
    if (a->relu_out) {
      if (pm == ROWS_DENSE) {
        d.relu = 0;  // the conv3 epilogue applies the ReLU after the residual add
      } else {
        d.relu = 1;
        d.relu_inactive_coarse = coarse;
      }
    }
    if ((rc = run_conv(&d, st))) return rc;
  } else if (a->out != a->x) {
    if ((rc = cuda_check(cudaMemcpyAsync(a->out, a->x, (size_t)n * ho * wo * a->c_out * (a->fp32 ? 4 : 2),
                                         cudaMemcpyDeviceToDevice, st),
                         "skip copy", 0)))
      return rc;
  }

  // ---------------------------------------------------------------- conv1 (unfused)
  if (conv1_done) {
  } else if (pm == ROWS_DENSE || (a->paradigm == LAUD_PARADIGM_SPATIAL && a->conv1_dense)) {
    c1.row_mode = ROWS_DENSE;
  } else if (a->paradigm == LAUD_PARADIGM_LAYER) {
    c1.row_mode = ROWS_PATCH;  // whole images of the active samples
    c1.list = cells;
    c1.count = cells_n;
    c1.patch_h = a->h_in;
    c1.patch_w = a->w_in;
    c1.cells_h = 1;
    c1.cells_w = 1;
  } else {
    if (!a->pix_list || !a->pix_count) return fail(LAUD_ERR_ARG, "pixel list workspace missing");
    if ((rc = laud_dilate_pixels(coarse, n, a->h_in, a->w_in, a->s, a->stride, 1, a->pix_list,
                                 a->pix_count, a->scan, stream)))
      return rc;
    c1.row_mode = ROWS_PIXEL;
    c1.list = a->pix_list;
    c1.count = a->pix_count;
  }
  if (!conv1_done && (rc = run_conv(&c1, st))) return rc;

  // ---------------------------------------------------------------- conv2 (3x3 over patches)
  laud_conv_args c2;
  memset(&c2, 0, sizeof(c2));
  c2.fp32 = a->fp32;
  c2.row_mode = pm2;
  c2.list = cells;
  c2.count = cells_n;
  c2.rows_max = n * ho * wo;
  c2.batch = n;
  c2.out_h = ho;
  c2.out_w = wo;
  c2.patch_h = ph;
  c2.patch_w = pw;
  c2.cells_h = ch;
  c2.cells_w = cw;
  c2.act = a->h1;
  c2.in_h = a->h_in;
  c2.in_w = a->w_in;
  c2.in_c = a->c_mid;
  c2.in_ld = a->c_mid;
  c2.ksize = 3;
  c2.stride = a->stride;
  c2.pad = 1;
  c2.weight = a->w2;
  c2.n_out = a->c_mid;
  c2.groups = a->groups;
  c2.latency_split = a->latency_split;
  // layer blocks (stride 1): conv2 / conv3 over the active samples' S x S
  // cells (the sample list expanded in the kernels) so conv2 runs on the halo
  // kernel instead of whole-image gathered rows; same K order, same result
  static const int lh_env = [] {
    const char* e = getenv("LAUD_LAYER_HALO");
    return e ? atoi(e) : 1;
  }();
  if (lh_env && a->paradigm == LAUD_PARADIGM_LAYER && a->stride == 1 && !a->fp32) {
    const int sl = a->c_mid <= 64 ? 4 : 2;
    if (ho % sl == 0 && wo % sl == 0) {
      c2.patch_h = c2.patch_w = sl;
      c2.cells_h = ho / sl;
      c2.cells_w = wo / sl;
      c2.list_expand = (ho / sl) * (wo / sl);
    }
  }
  c2.scale = a->s2;
  c2.bias = a->b2;
  c2.relu = a->relu2;
  c2.out_mode = OUT_ROW;
  c2.out = a->h2;
  c2.out_ld = a->c_mid;
  if ((rc = run_conv(&c2, st))) return rc;
  if (a->se_w1) {  // EXT squeeze-excitation over each sample's conv2 rows
    if (a->fp32) return fail(LAUD_ERR_UNSUPPORTED, "SE in fp32 mode");
    if (!a->se_b1 || !a->se_w2 || !a->se_b2 || a->se_hidden < 1)
      return fail(LAUD_ERR_ARG, "SE weights incomplete");
    ProfScope ps(3, st);
    if ((rc = cuda_check(launch_se(a->h2, n, a->c_mid, pm == ROWS_DENSE ? nullptr : cells,
                                   pm == ROWS_DENSE ? nullptr : cells_n, ch * cw, ph * pw, ho * wo,
                                   a->se_w1, a->se_b1, a->se_hidden, a->se_w2, a->se_b2, a->h1, st),
                         "se", 3)))
      return rc;
  }

  // ---------------------------------------------------------------- conv3 + scatter-add
  laud_conv_args c3 = c2;
  c3.groups = 1;
  c3.act = a->h2;
  c3.in_h = ho;
  c3.in_w = wo;
  c3.a_compact = 1;
  c3.ksize = 1;
  c3.stride = 1;
  c3.pad = 0;
  c3.weight = a->w3;
  c3.n_out = a->c_out;
  c3.scale = a->s3;
  c3.bias = a->b3;
  c3.relu = a->relu_out;
  c3.out_mode = OUT_PIXEL;
  c3.out = a->out;
  c3.out_ld = a->c_out;
  c3.resid = a->out;
  c3.resid_ld = a->c_out;
  c3.misplace_first = a->misplace_first;
  if (a->next_wdiff && a->dn && pm == ROWS_PATCH) {  // dot with the next block's masker
    c3.mdot_w = a->next_wdiff;
    c3.mdot_out = a->dn;
  }
  return run_conv(&c3, st);
}

int laud_stem_im2col(const uint8_t* img, int n, int h, int w, int k, int stride, int pad,
                     const float* mean, const float* inv_std, void* cols, int cols_ld,
                     void* stream) {
  if ((k != 3 && k != 7) || cols_ld != k * ((k * 3 + 7) / 8 * 8))
    return fail(LAUD_ERR_SHAPE, "stem im2col: k must be 3 or 7 and cols_ld = k * pad8(3k)");
  ProfScope ps(3, (cudaStream_t)stream);
  return cuda_check(launch_stem_im2col(img, n, h, w, k, stride, pad, mean, inv_std, cols, cols_ld,
                                       (cudaStream_t)stream),
                    "stem im2col", 1);
}

int laud_maxpool3s2(const void* x, int n, int h, int w, int c, void* y, void* stream) {
  if (c % 8) return fail(LAUD_ERR_SHAPE, "channels must be a multiple of 8");
  ProfScope ps(3, (cudaStream_t)stream);
  return cuda_check(launch_maxpool3s2(x, n, h, w, c, y, (cudaStream_t)stream), "maxpool", 1);
}

int laud_stem_pool(const uint8_t* img, int n, int h, int w, const float* mean, const float* inv_std,
                   const void* weight, const float* bias, void* out, void* stream) {
  if (!img || !mean || !inv_std || !weight || !bias || !out) return fail(LAUD_ERR_ARG, "null pointer in stem args");
  if (h != 224 || w != 224) return fail(LAUD_ERR_SHAPE, "fused stem: 224x224 images (got %dx%d)", h, w);
  if (n <= 0) return LAUD_OK;
  if ((reinterpret_cast<uintptr_t>(weight) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(LAUD_ERR_ARG, "fused stem: 16-byte aligned weights and output");
  ProfScope ps(3, (cudaStream_t)stream);
  return cuda_check(launch_stem_pool(img, n, mean, inv_std, weight, bias, out, num_sms(), (cudaStream_t)stream),
                    "fused stem", 1);
}

int laud_stem3(const uint8_t* img, int n, int h, int w, const float* mean, const float* inv_std,
               const void* weight, const float* bias, void* out, void* stream) {
  if (!img || !mean || !inv_std || !weight || !bias || !out) return fail(LAUD_ERR_ARG, "null pointer in stem args");
  if (h != 224 || w != 224) return fail(LAUD_ERR_SHAPE, "fused 3x3 stem: 224x224 images (got %dx%d)", h, w);
  if (n <= 0) return LAUD_OK;
  if ((reinterpret_cast<uintptr_t>(weight) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(LAUD_ERR_ARG, "fused 3x3 stem: 16-byte aligned weights and output");
  ProfScope ps(3, (cudaStream_t)stream);
  return cuda_check(launch_stem3(img, n, mean, inv_std, weight, bias, out, num_sms(), (cudaStream_t)stream),
                    "fused 3x3 stem", 1);
}

int laud_global_avgpool(const void* x, int n, int hw, int c, void* y, void* stream) {
  ProfScope ps(3, (cudaStream_t)stream);
  return cuda_check(launch_gap(x, n, hw, c, y, (cudaStream_t)stream), "global avgpool", 1);
}

}  // extern "C"
