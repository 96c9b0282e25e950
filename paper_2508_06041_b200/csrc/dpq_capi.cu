// Host side of libdpq_b200.so: handles, device memory, op descriptors, the
// per-step kernel schedule and its CUDA graph. C-ABI in include/dpq_b200.h.
#include "dpq_kernels.cu"
#include "dpq_engine.cu"
#include "dpq_gemv.cu"

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <utility>
#include <algorithm>
#include <vector>

#include "../../include/dpq_b200.h"

using namespace dpq;

namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return set_err(DPQ_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                     __FILE__, __LINE__);                                                \
  } while (0)

#define TRY(expr)              \
  do {                         \
    int r_ = (expr);           \
    if (r_ != DPQ_OK) return r_; \
  } while (0)

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

constexpr int kOpSmemAlloc = (int)kLutShared + kLutBytes;   // covers any dynamic base >= 0

// Device allocations owned by a handle.
struct Arena {
  std::vector<void*> ptrs;
  int alloc(void** p, size_t bytes) {
    if (bytes == 0) bytes = 16;
    CK(cudaMalloc(p, bytes));
    CK(cudaMemset(*p, 0, bytes));
    ptrs.push_back(*p);
    return DPQ_OK;
  }
  template <typename T>
  int alloc_t(T** p, size_t n) {
    return alloc(reinterpret_cast<void**>(p), n * sizeof(T));
  }
  void release() {
    for (void* p : ptrs) cudaFree(p);
    ptrs.clear();
  }
};

struct Scratch {
  float* part = nullptr;
  float* part_lo = nullptr;
  float* gx_part = nullptr;
  double* win_stats = nullptr;
  float* op_stats = nullptr;
  unsigned* tile_cnt = nullptr;
  float* out_lo = nullptr;
  float* out_hi = nullptr;
  float* dual_sq = nullptr;
  size_t part_elems = 0, tiles = 0, rows = 0;
  int n_win = 0;
  int make(Arena& a, int n_win_max, size_t rows_pad_max, size_t tiles_max) {
    n_win = n_win_max;
    part_elems = (size_t)n_win_max * rows_pad_max;
    tiles = tiles_max;
    rows = rows_pad_max;
    TRY(a.alloc_t(&part, part_elems));
    TRY(a.alloc_t(&part_lo, part_elems));
    TRY(a.alloc_t(&gx_part, (size_t)kMaxOpLayers * n_win_max * kMaxK));
    TRY(a.alloc_t(&win_stats, (size_t)4 * n_win_max));
    TRY(a.alloc_t(&op_stats, 4));
    TRY(a.alloc_t(&tile_cnt, tiles_max));
    TRY(a.alloc_t(&out_lo, rows_pad_max));
    TRY(a.alloc_t(&out_hi, rows_pad_max));
    TRY(a.alloc_t(&dual_sq, tiles_max));
    return DPQ_OK;
  }
  void fill(OpDesc& D) const {
    D.part = part;
    D.part_lo = part_lo;
    D.gx_part = gx_part;
    D.win_stats = win_stats;
    D.op_stats = op_stats;
    D.tile_cnt = tile_cnt;
    D.out_lo = out_lo;
    D.out_hi = out_hi;
    D.dual_sq = dual_sq;
  }
};

int g_n_sm = -1;

int num_sms(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return 148;
  return n;
}

bool g_attr_done = false;
int set_kernel_attrs() {
  if (g_attr_done) return DPQ_OK;
  CK(cudaFuncSetAttribute(op_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kOpSmemAlloc));
  g_attr_done = true;
  return DPQ_OK;
}

// Launch helper: cudaLaunchKernelEx with optional programmatic serialization.
template <typename... KArgs, typename... Args>
int launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
           Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  if (pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  CK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
  return DPQ_OK;
}

// Grid of an op: every window needs >= 1 CTA, never more CTAs than SMs
// (the decision barrier needs all CTAs co-resident: 1 CTA/SM by smem).
// Tile CTAs of an op (one SM is reserved for the op's decider CTA).
int op_grid(const OpDesc& D, int n_sm) {
  long long units = (long long)D.n_win * D.total_tiles;
  int g = (int)std::min<long long>(units, n_sm - 1);
  return std::max(g, D.n_win);
}

}  // namespace

// ---------------------------------------------------------------------------
// handles
// ---------------------------------------------------------------------------
struct dpq_store {
  int device = 0;
  int n_sm = 148;
  std::vector<DevLayer> layers;
  std::vector<float*> hi;            // device copies of hi (dequantize)
  std::vector<long long> plane_bytes;
  Arena arena;
  // standalone-op state
  Scratch scratch;
  Control* ctl = nullptr;
  OpSync* sync = nullptr;
  unsigned* ctr = nullptr;
  long long* gxa = nullptr;
  int* decision = nullptr;
  signed char* tr_bits = nullptr;
  float* tr_est = nullptr;
  float* tr_exact = nullptr;
  float* est_buf = nullptr;          // exact-estimator input copy
  int max_rows_pad = 0, max_win = 0, max_tiles = 0, max_cols = 0;
  std::vector<void*> gemv_progs;     // single-op engine programs per layer (dpq_gemv)
  // bitplane_gemv_kernel scratch (dpq_gemv.cu; self-resetting, sized for the largest layer seen)
  Arena gv_arena;
  gv::Args gv{};
  size_t gv_part = 0, gv_tiles = 0, gv_win = 0;
  int gv_smem = 0;
};

struct dpq_plan {
  dpq_store* store = nullptr;
  std::vector<DevSel> sel;
  std::vector<dpq_sel_desc> host;    // copy of the descriptors (G pointers cleared)
  Arena arena;
  int any_prev = 0;
  std::vector<int> gt_fb;            // per layer: fixed-point fraction bits of the engine's G.x sums
  std::vector<void*> gemv_progs;     // single-op engine programs per layer (dpq_select_gemv)
};

int gemv_engine_run(dpq_store* s, dpq_plan* p, int li, int b, const float* x, float* y, int32_t* bit_out,
                    float* est_out, cudaStream_t st, bool* used);

// One layer through bitplane_gemv_kernel (dpq_gemv.cu): static b (p == nullptr)
// or the plan's selector. *used = false when the layer does not fit it (a CTA
// range over > 2 windows, an exact estimator): the caller falls back.
int gv_run(dpq_store* s, const dpq_plan* p, int li, int b, const float* x, float* y, int32_t* bit_out,
           float* est_out, cudaStream_t st, bool* used) {
  *used = false;
  const char* env = getenv("DPQ_GEMV_KERNEL");
  if (env && env[0] == '0') return DPQ_OK;
  const DevLayer& L = s->layers[li];
  const long long T = (long long)L.n_win * L.n_tiles;
  const int G = (int)std::min<long long>(s->n_sm, T);
  if (G <= 0 || (T + G - 1) / G > L.n_tiles + 1) return DPQ_OK;      // <= 2 windows per CTA
  gv::Args A{};
  A.l = A.h = b;
  A.sentinel = 1;
  if (p) {
    const DevSel& S = p->sel[li];
    if (S.sentinel == 0 && S.est_kind != EST_LINEAR && !(S.est_kind == EST_PROJECTION && S.G && S.k <= kMaxK))
      return DPQ_OK;
    // the selector here decides after the base planes are issued and streams the
    // extra planes at the end (their latency is exposed); the single-op engine
    // program overlaps them, which wins once the base stream is long
    // (tools/gemv_sweep.py: 4096x4096 13.7 vs 16.6 us, 14336x4096 21.6 vs 20.6)
    const char* dyn_env = getenv("DPQ_GEMV_KERNEL_DYNAMIC");
    const long long max_dyn = dyn_env ? atoll(dyn_env) : (1ll << 62);
    if (S.l != S.h && (long long)L.rows * L.cols * S.l / 8 > max_dyn) return DPQ_OK;
    A.l = S.l;
    A.h = S.h;
    A.sentinel = S.sentinel;
    A.est_kind = S.est_kind;
    A.k = S.est_kind == EST_PROJECTION ? S.k : 0;
    A.g_dtype = S.g_dtype;
    A.G = S.G;
    A.g_scale = S.g_scale;
    A.T = S.T;
    A.slope = S.slope;
    A.intercept = S.intercept;
    A.fbscale = std::ldexp(1.0, -p->gt_fb[li]);
    A.fxscale = std::ldexp(1.0, p->gt_fb[li]);
    if (A.l == A.h) A.sentinel = 1;
  }
  const size_t part = (size_t)L.n_win * L.n_tiles * 32;
  if (part > s->gv_part || (size_t)L.n_tiles > s->gv_tiles || (size_t)L.n_win > s->gv_win || !s->gv.sync) {
    CK(cudaStreamSynchronize(st));
    s->gv_arena.release();
    s->gv_part = std::max(part, s->gv_part);
    s->gv_tiles = std::max((size_t)L.n_tiles, s->gv_tiles);
    s->gv_win = std::max((size_t)L.n_win, s->gv_win);
    gv::Args& S = s->gv;
    TRY(s->gv_arena.alloc_t(&S.part, s->gv_part));
    TRY(s->gv_arena.alloc_t(&S.cnt, s->gv_tiles));
    TRY(s->gv_arena.alloc_t(&S.sx, s->gv_win));
    TRY(s->gv_arena.alloc_t(&S.sq, s->gv_win));
    TRY(s->gv_arena.alloc_t(&S.acc, (size_t)kMaxK));
    TRY(s->gv_arena.alloc_t(&S.sync, 4));
    TRY(s->gv_arena.alloc_t(&S.err, 1));
  }
  if (!s->gv_smem) {
    int optin = 0;
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, s->device));
    s->gv_smem = optin - 1024;
    CK(cudaFuncSetAttribute(gv::bitplane_gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, s->gv_smem));
  }
  A.part = s->gv.part;
  A.cnt = s->gv.cnt;
  A.sx = s->gv.sx;
  A.sq = s->gv.sq;
  A.acc = s->gv.acc;
  A.sync = s->gv.sync;
  A.err = s->gv.err;
  A.planes = L.planes;
  A.pstride16 = L.plane_stride16;
  A.lo = L.lo;
  A.span = L.span;
  A.rows = L.rows;
  A.cols = L.cols;
  A.n_win = L.n_win;
  A.n_tiles = L.n_tiles;
  A.x = x;
  A.y = y;
  A.bit_out = bit_out;
  A.est_out = est_out;
  const char* pdl_env = getenv("DPQ_GEMV_PDL");
  const bool pdl = !(pdl_env && pdl_env[0] == '0');
  TRY(launch(gv::bitplane_gemv_kernel, dim3(G), dim3(gv::kNT), (size_t)s->gv_smem, st, pdl, A));
  *used = true;
  return DPQ_OK;
}
void gemv_progs_release(std::vector<void*>& cache);


struct OpStep {
  enum Kind { OP, FINALIZE, DECIDE_EXACT, PREP_EST } kind;
  OpDesc desc;
  int grid;
};

struct dpq_session {
  dpq_store* store = nullptr;
  dpq_plan* plan = nullptr;
  dpq_model_desc m{};
  int n_sm = 148;
  cudaStream_t stream = nullptr;
  Arena arena;
  Control* ctl = nullptr;
  Control* ctl_host = nullptr;       // pinned staging for the host-written fields
  unsigned char* pin_io = nullptr;   // pinned per-step staging (dpq_session_step): control words in,
                                     // logits + error flags out
  signed char* forced_dev = nullptr;
  float *x = nullptr, *qkv = nullptr, *attn = nullptr, *ug = nullptr, *logits = nullptr;
  float *embed = nullptr, *lm = nullptr, *cosv = nullptr, *sinv = nullptr;
  std::vector<float*> kc, vc;
  float* attn_part = nullptr;
  unsigned* attn_cnt = nullptr;
  unsigned* head_cnt = nullptr;
  int* tok_log = nullptr;
  float* est_x = nullptr;            // exact-with-previous-input estimator input
  Scratch scratch;
  OpSync* syncs = nullptr;
  unsigned* ctrs = nullptr;
  long long* gxas = nullptr;
  int* decisions = nullptr;
  float *snap = nullptr, *snap_stats = nullptr;
  signed char* tr_bits = nullptr;
  float *tr_est = nullptr, *tr_exact = nullptr;
  int n_trace = 0, max_steps = 0, n_chunks = 0;
  std::vector<OpStep> sched;         // per block ops in execution order
  std::vector<AttnDesc> attn_desc;
  HeadDesc head{};
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  int pos_host = 0;
  int steps_host = 0;
  unsigned long long* dbg = nullptr;
  int dbg_per_op = 0;
  // persistent step kernel
  bool persistent = false;
  Scratch scratch2;                  // ping-pong scratch (ops alternate)
  unsigned* flags = nullptr;
  size_t n_flags = 0;
  StepDesc step{};
  std::vector<OpDesc> ops;           // main ops in execution order
  // persistent decode engine (dpq_engine.cu)
  bool engine = false;
  eng::Prog prog{};
  eng::ECtl* ectl = nullptr;
  float* h = nullptr;
  int eng_smem = 0;
  int eng_grid = 0;
  unsigned long long* eng_dbg = nullptr;
  std::vector<unsigned long long*> eng_vec;   // tagged vectors (reset to "no epoch")
  std::vector<size_t> eng_vec_len;
  size_t eng_fpart_len = 0;         // tagged estimator-set words (engine)
  // tensor parallelism (row shards over tp_size ranks; dpq_session_create_tp)
  int tp_size = 1, tp_rank = 0;
  void* xarena = nullptr;           // exchange arena (cudaMalloc: one IPC handle)
  size_t xarena_bytes = 0;
};

// ---------------------------------------------------------------------------
// layout reference (host) — used by tests, mirrors repack_kernel
// ---------------------------------------------------------------------------
extern "C" int64_t dpq_planes_bytes(int rows, int cols, int n_bits) {
  const long long n_tiles = cdiv(rows, kTileRows), n_win = cdiv(cols, kWinCols);
  return (int64_t)n_bits * n_win * n_tiles * kTileBytes;
}

extern "C" int dpq_repack_host(const uint16_t* codes, int rows, int cols, int n_bits, uint8_t* planes,
                               int64_t planes_bytes) {
  if (!codes || !planes || rows < 1 || cols < 1 || n_bits < 1 || n_bits > 8)
    return set_err(DPQ_ERR_ARG, "dpq_repack_host: bad arguments");
  const int n_tiles = cdiv(rows, kTileRows), n_win = cdiv(cols, kWinCols);
  if (planes_bytes < dpq_planes_bytes(rows, cols, n_bits))
    return set_err(DPQ_ERR_ARG, "dpq_repack_host: output too small");
  for (int row = 0; row < n_tiles * 32; ++row)
    for (int w = 0; w < n_win; ++w)
      for (int g = 0; g < kGroups; ++g) {
        const int tile = row >> 5, lane = row & 31;
        const int s = (g - lane + 64) & 63;
        const int wrap = (lane + s) >= 64;
        for (int p = 0; p < n_bits; ++p) {
          unsigned e = 0;
          for (int t = 0; t < 8; ++t) {
            const int col = w * kWinCols + 8 * g + t;
            unsigned c = (row < rows && col < cols) ? codes[(size_t)row * cols + col] : 0u;
            e |= ((c >> (n_bits - 1 - p)) & 1u) << t;
          }
          e = (e - wrap) & 255u;
          const long long off = (((long long)p * n_win + w) * n_tiles + tile) * kTileBytes +
                                (s >> 4) * 512 + lane * 16 + (s & 15);
          planes[off] = (uint8_t)e;
        }
      }
  return DPQ_OK;
}

// ---------------------------------------------------------------------------
// misc
// ---------------------------------------------------------------------------
static unsigned long long* g_diag_host = nullptr;   // mapped: engine watchdog record
static int* g_prog_host = nullptr;                    // mapped: per-CTA progress (DPQ_ENGINE_TRACE)

extern "C" const char* dpq_last_error(void) {
  if (g_diag_host && g_diag_host[0]) {
    char buf[512];
    snprintf(buf, sizeof(buf), " [engine watchdog: dpq_engine.cu line %llu, block %llu, thread %llu, args %lld %lld"
             " extra %llx %llx %llx %llx %llx %llx]",
             g_diag_host[1], g_diag_host[2], g_diag_host[3], (long long)g_diag_host[4], (long long)g_diag_host[5],
             g_diag_host[6], g_diag_host[7], g_diag_host[8], g_diag_host[9], g_diag_host[10], g_diag_host[11]);
    g_err += buf;
    g_err += " wstate:";
    for (int q = 0; q < 16; ++q) {
      snprintf(buf, sizeof(buf), " %llu/%llu", g_diag_host[12 + q] / 16, g_diag_host[12 + q] % 16);
      g_err += buf;
    }
    g_diag_host[0] = 0;
    if (g_prog_host) {
      std::string pr = " progress(cta: step<<16|stage, phase, prod_j, prod_op):";
      for (int c = 0; c < 148; ++c) {
        snprintf(buf, sizeof(buf), " %d:%x,%d,%d,%d", c, g_prog_host[4 * c], g_prog_host[4 * c + 1], g_prog_host[4 * c + 2],
                 g_prog_host[4 * c + 3]);
        pr += buf;
      }
      g_err += pr;
    }
  }
  return g_err.c_str();
}
extern "C" int dpq_version(void) { return 1; }

extern "C" int dpq_device_info(int device, int* n_sm, int* cc_major, int* cc_minor) {
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return set_err(DPQ_ERR_ARG, "no CUDA device %d", device);
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (n_sm) *n_sm = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  return DPQ_OK;
}

extern "C" int dpq_quantize_device(int device, const float* W_dev, int rows, int cols, int n_bits,
                                   uint16_t* codes_dev, float* lo_dev, float* hi_dev, void* stream) {
  if (rows < 1 || cols < 1 || n_bits < 2 || n_bits > 8)
    return set_err(DPQ_ERR_ARG, "dpq_quantize_device: bad shape/bits");
  CK(cudaSetDevice(device));
  quantize_kernel<<<rows, 256, 0, (cudaStream_t)stream>>>(W_dev, rows, cols, n_bits, codes_dev, lo_dev,
                                                          hi_dev);
  CK(cudaGetLastError());
  return DPQ_OK;
}

// ---------------------------------------------------------------------------
// store
// ---------------------------------------------------------------------------
// One layer: codes (host or device; uint16 / uint8 / the .dpqs packed stream)
// repacked into bitplanes on the device; lo / span / hi padded to whole tiles.
static int store_add_layer(dpq_store* s, const dpq_layer_desc& d, int i) {
  if (d.rows < 1 || d.cols < 1 || d.n_bits < 2 || d.n_bits > 8 || d.b_min < 1 || d.b_min > d.n_bits ||
      (d.code_bytes < 0 || d.code_bytes > 2) || !d.codes || !d.lo || !d.hi)
    return set_err(DPQ_ERR_ARG, "dpq_store_create: bad layer %d", i);
  DevLayer L{};
  L.rows = d.rows;
  L.cols = d.cols;
  L.n_bits = d.n_bits;
  L.b_min = d.b_min;
  L.n_tiles = cdiv(d.rows, kTileRows);
  L.n_win = cdiv(d.cols, kWinCols);
  L.plane_stride16 = (long long)L.n_win * L.n_tiles * (kTileBytes / 16);
  const long long pbytes = dpq_planes_bytes(d.rows, d.cols, d.n_bits);
  void* planes = nullptr;
  if (s->arena.alloc(&planes, pbytes)) return DPQ_ERR_CUDA;
  const void* codes_dev = d.codes;
  void* tmp = nullptr;
  const size_t cbytes = d.code_bytes ? (size_t)d.rows * d.cols * d.code_bytes
                                     : ((size_t)d.rows * d.cols * d.n_bits + 7) / 8;   // .dpqs packed
  if (!d.codes_on_device) {
    if (cudaMalloc(&tmp, cbytes) != cudaSuccess ||
        cudaMemcpy(tmp, d.codes, cbytes, cudaMemcpyHostToDevice) != cudaSuccess) {
      if (tmp) cudaFree(tmp);
      return set_err(DPQ_ERR_CUDA, "dpq_store_create: code upload failed");
    }
    codes_dev = tmp;
  }
  const long long groups = (long long)L.n_tiles * 32 * L.n_win * kGroups;
  const int blocks = (int)std::min<long long>((groups + 255) / 256, 65535LL * 16);
  repack_kernel<<<blocks, 256>>>(codes_dev, d.code_bytes, d.rows, d.cols, d.n_bits, L.n_win, L.n_tiles,
                                 reinterpret_cast<unsigned char*>(planes));
  cudaError_t e = cudaDeviceSynchronize();
  if (tmp) cudaFree(tmp);
  if (e != cudaSuccess) return set_err(DPQ_ERR_CUDA, "repack: %s", cudaGetErrorString(e));
  L.planes = reinterpret_cast<const uint4*>(planes);
  const int rp = L.n_tiles * 32;
  std::vector<float> lo(rp, 0.f), span(rp, 0.f), hi(rp, 0.f);
  for (int r = 0; r < d.rows; ++r) {
    lo[r] = d.lo[r];
    hi[r] = d.hi[r];
    span[r] = (float)((double)d.hi[r] - (double)d.lo[r]);
  }
  float *dlo, *dspan, *dhi;
  if (s->arena.alloc_t(&dlo, rp) || s->arena.alloc_t(&dspan, rp) || s->arena.alloc_t(&dhi, rp))
    return DPQ_ERR_CUDA;
  if (cudaMemcpy(dlo, lo.data(), rp * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(dspan, span.data(), rp * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(dhi, hi.data(), rp * 4, cudaMemcpyHostToDevice) != cudaSuccess)
    return set_err(DPQ_ERR_CUDA, "dpq_store_create: lo/hi upload failed");
  L.lo = dlo;
  L.span = dspan;
  s->layers.push_back(L);
  s->hi.push_back(dhi);
  s->plane_bytes.push_back(pbytes);
  return DPQ_OK;
}

// Standalone-op scratch for the store's current largest layer (re-made when
// appended layers grow it; the old scratch stays in the arena).
static int store_make_scratch(dpq_store* s) {
  int rp = 32, nw = 1, nt = 1, nc = 1;
  for (const DevLayer& L : s->layers) {
    rp = std::max(rp, L.n_tiles * 32);
    nw = std::max(nw, L.n_win);
    nt = std::max(nt, L.n_tiles);
    nc = std::max(nc, L.cols);
  }
  if (s->ctl && rp <= s->max_rows_pad && nw <= s->max_win && nt <= s->max_tiles && nc <= s->max_cols) return DPQ_OK;
  s->max_rows_pad = rp;
  s->max_win = nw;
  s->max_tiles = nt;
  s->max_cols = nc;
  if (s->scratch.make(s->arena, s->max_win, s->max_rows_pad, s->max_tiles) ||
      s->arena.alloc_t(&s->ctl, 1) || s->arena.alloc_t(&s->sync, 2) || s->arena.alloc_t(&s->decision, 4) ||
      s->arena.alloc_t(&s->ctr, 128) || s->arena.alloc_t(&s->gxa, kMaxOpLayers * kMaxK) ||
      s->arena.alloc_t(&s->tr_bits, 4) || s->arena.alloc_t(&s->tr_est, 4) ||
      s->arena.alloc_t(&s->tr_exact, 4) || s->arena.alloc_t(&s->est_buf, s->max_cols))
    return DPQ_ERR_CUDA;
  Control c{};
  c.mode = MODE_DYNAMIC;
  if (cudaMemcpy(s->ctl, &c, sizeof(c), cudaMemcpyHostToDevice) != cudaSuccess)
    return set_err(DPQ_ERR_CUDA, "dpq_store_create: control init failed");
  return DPQ_OK;
}

extern "C" int dpq_store_create(int device, int n_layers, const dpq_layer_desc* descs, dpq_store** out) {
  if (!out || n_layers < 0 || (n_layers > 0 && !descs)) return set_err(DPQ_ERR_ARG, "dpq_store_create: bad arguments");
  *out = nullptr;
  CK(cudaSetDevice(device));
  TRY(set_kernel_attrs());
  dpq_store* s = new dpq_store();
  s->device = device;
  s->n_sm = num_sms(device);
  auto fail = [&](int code) {
    s->arena.release();
    delete s;
    return code;
  };
  for (int i = 0; i < n_layers; ++i) {
    const int r = store_add_layer(s, descs[i], i);
    if (r != DPQ_OK) return fail(r);
  }
  if (n_layers > 0) {
    const int r = store_make_scratch(s);
    if (r != DPQ_OK) return fail(r);
  }
  *out = s;
  return DPQ_OK;
}

extern "C" int dpq_store_append(dpq_store* s, int n_layers, const dpq_layer_desc* descs) {
  if (!s || n_layers < 1 || !descs) return set_err(DPQ_ERR_ARG, "dpq_store_append: bad arguments");
  CK(cudaSetDevice(s->device));
  for (int i = 0; i < n_layers; ++i) TRY(store_add_layer(s, descs[i], (int)s->layers.size()));
  return store_make_scratch(s);
}

extern "C" int dpq_store_destroy(dpq_store* s) {
  if (!s) return DPQ_OK;
  cudaSetDevice(s->device);
  cudaDeviceSynchronize();
  gemv_progs_release(s->gemv_progs);
  s->gv_arena.release();
  s->arena.release();
  delete s;
  return DPQ_OK;
}

extern "C" int dpq_store_layer_bytes(const dpq_store* s, int layer, int b, int64_t* bytes) {
  if (!s || layer < 0 || layer >= (int)s->layers.size() || !bytes)
    return set_err(DPQ_ERR_ARG, "dpq_store_layer_bytes: bad arguments");
  const DevLayer& L = s->layers[layer];
  *bytes = (int64_t)L.rows * L.cols * b / 8 + 8LL * L.rows + 4LL * L.cols + 4LL * L.rows;
  return DPQ_OK;
}

namespace {

// Single-layer op on the store's private scratch.
OpDesc single_op(dpq_store* s, int layer, const DevSel& S, const float* x, float* y) {
  OpDesc D{};
  const DevLayer& L = s->layers[layer];
  D.n_layers = 1;
  D.cols = L.cols;
  D.n_win = L.n_win;
  D.total_tiles = L.n_tiles;
  D.rows_total_pad = L.n_tiles * 32;
  D.in_mode = IN_IDENT;
  D.out_mode = OUT_STORE;
  D.eps = 1e-6f;
  D.in0 = x;
  D.out = y;
  s->scratch.fill(D);
  D.decision = s->decision;
  D.main_decision = s->decision;
  D.sync = s->sync;
  D.ctr = s->ctr;
  D.gxa = s->gxa;
  D.tr_bits = s->tr_bits;
  D.tr_est = s->tr_est;
  D.tr_exact = s->tr_exact;
  D.n_trace = 1;
  D.max_steps = 1;
  D.layer[0].L = L;
  D.layer[0].S = S;
  D.layer[0].trace_idx = 0;
  D.layer[0].snap_in = -1;
  return D;
}

__global__ void copy_sel_outputs(const signed char* bits, const float* est, const float* exact,
                                 int32_t* bit_out, float* est_out, float* exact_out) {
  if (threadIdx.x == 0) {
    if (bit_out) *bit_out = bits[0];
    if (est_out) *est_out = est[0];
    if (exact_out) *exact_out = exact[0];
  }
}

__global__ void reset_trace1(signed char* bits, float* est, float* exact) {
  if (threadIdx.x == 0) {
    bits[0] = -1;
    est[0] = CUDART_NAN_F;
    exact[0] = CUDART_NAN_F;
  }
}

int run_op(const OpDesc& D, Control* ctl, int n_sm, cudaStream_t st, bool pdl) {
  const int g = op_grid(D, n_sm) + 1;      // + the decider CTA
  return launch(op_kernel, dim3(g), dim3(kThreads), (size_t)kOpSmemAlloc, st, pdl, D, ctl);
}

}  // namespace

// Diagnostics (not in the public header): per-CTA globaltimer stamps of
// bitplane_gemv_kernel into dev_buf [grid][8] (nullptr: off). tools/gv_stamps.py.
extern "C" int dpq_debug_gemv_stamps(unsigned long long* dev_buf) {
  CK(cudaMemcpyToSymbol(gv::g_gv_dbg, &dev_buf, sizeof(dev_buf)));
  return DPQ_OK;
}

extern "C" int dpq_gemv(dpq_store* s, int layer, int b, const float* x_dev, float* y_dev, void* stream) {
  if (!s || layer < 0 || layer >= (int)s->layers.size() || !x_dev || !y_dev)
    return set_err(DPQ_ERR_ARG, "dpq_gemv: bad arguments");
  const DevLayer& L = s->layers[layer];
  if (b < L.b_min || b > L.n_bits)
    return set_err(DPQ_ERR_ARG, "bitwidth %d outside [%d, %d]", b, L.b_min, L.n_bits);
  CK(cudaSetDevice(s->device));
  DevSel S{};
  S.l = S.h = S.prefill_bit = b;
  S.sentinel = 1;
  S.T = INFINITY;
  bool used = false;
  TRY(gv_run(s, nullptr, layer, b, x_dev, y_dev, nullptr, nullptr, (cudaStream_t)stream, &used));
  if (used) return DPQ_OK;
  TRY(gemv_engine_run(s, nullptr, layer, b, x_dev, y_dev, nullptr, nullptr, (cudaStream_t)stream, &used));
  if (used) return DPQ_OK;
  OpDesc D = single_op(s, layer, S, x_dev, y_dev);
  D.layer[0].trace_idx = -1;
  D.n_trace = 0;
  return run_op(D, s->ctl, s->n_sm, (cudaStream_t)stream, false);
}

extern "C" int dpq_dequantize(dpq_store* s, int layer, int b, double* out_dev, void* stream) {
  if (!s || layer < 0 || layer >= (int)s->layers.size() || !out_dev)
    return set_err(DPQ_ERR_ARG, "dpq_dequantize: bad arguments");
  const DevLayer& L = s->layers[layer];
  if (b < L.b_min || b > L.n_bits)
    return set_err(DPQ_ERR_ARG, "bitwidth %d outside [%d, %d]", b, L.b_min, L.n_bits);
  CK(cudaSetDevice(s->device));
  const long long n = (long long)L.rows * L.cols;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 65535LL * 8);
  dequant_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(L, s->hi[layer], b, out_dev);
  CK(cudaGetLastError());
  return DPQ_OK;
}

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------
extern "C" int dpq_plan_create(dpq_store* s, int n_layers, const dpq_sel_desc* sels, dpq_plan** out) {
  if (!s || !sels || !out || n_layers != (int)s->layers.size())
    return set_err(DPQ_ERR_ARG, "dpq_plan_create: need one selector per store layer");
  *out = nullptr;
  CK(cudaSetDevice(s->device));
  dpq_plan* p = new dpq_plan();
  p->store = s;
  auto fail = [&](int code) {
    p->arena.release();
    delete p;
    return code;
  };
  for (int i = 0; i < n_layers; ++i) {
    const dpq_sel_desc& d = sels[i];
    const DevLayer& L = s->layers[i];
    DevSel S{};
    S.l = d.l;
    S.h = d.h;
    S.prefill_bit = d.prefill_bit;
    S.T = d.T;
    S.sentinel = std::isinf(d.T) ? (d.T > 0 ? 1 : 2) : 0;
    S.est_kind = d.est_kind;
    S.prev_residual = d.prev_residual;
    S.slope = d.slope;
    S.intercept = d.intercept;
    S.k = d.k;
    S.g_dtype = d.g_dtype;
    for (int b : {d.l, d.h, d.prefill_bit})
      if (b < L.b_min || b > L.n_bits)
        return fail(set_err(DPQ_ERR_ARG, "layer %d: bitwidth %d outside [%d, %d]", i, b, L.b_min, L.n_bits));
    if (S.sentinel == 0 && d.est_kind == EST_NONE)
      return fail(set_err(DPQ_ERR_ARG, "layer %d: finite threshold needs an estimator", i));
    if (S.sentinel == 0 && d.est_kind == EST_PROJECTION) {
      if (d.k < 1 || d.k > kMaxK || !d.G)
        return fail(set_err(DPQ_ERR_ARG, "layer %d: projection rank %d outside [1, %d]", i, d.k, kMaxK));
      // [k][cols] fp64 -> [n_win][k][512] in g_dtype (+ per-row scale for e4m3)
      const size_t n = (size_t)L.n_win * d.k * kWinCols;
      std::vector<float> rowscale(d.k, 1.f);
      if (d.g_dtype == G_E4M3) {
        for (int r = 0; r < d.k; ++r) {
          double mx = 0.0;
          for (int c = 0; c < L.cols; ++c) mx = std::max(mx, std::fabs(d.G[(size_t)r * L.cols + c]));
          rowscale[r] = mx > 0.0 ? (float)(mx / 448.0) : 1.f;
        }
      }
      auto src = [&](int w, int r, int c) -> double {
        const int col = w * kWinCols + c;
        if (col >= L.cols) return 0.0;
        return d.G[(size_t)r * L.cols + col];
      };
      void* gdev = nullptr;
      if (d.g_dtype == G_F32) {
        std::vector<float> h(n);
        for (int w = 0; w < L.n_win; ++w)
          for (int r = 0; r < d.k; ++r)
            for (int c = 0; c < kWinCols; ++c) h[((size_t)w * d.k + r) * kWinCols + c] = (float)src(w, r, c);
        if (p->arena.alloc(&gdev, n * 4) || cudaMemcpy(gdev, h.data(), n * 4, cudaMemcpyHostToDevice))
          return fail(set_err(DPQ_ERR_CUDA, "G upload"));
      } else if (d.g_dtype == G_F16) {
        std::vector<__half> h(n);
        for (int w = 0; w < L.n_win; ++w)
          for (int r = 0; r < d.k; ++r)
            for (int c = 0; c < kWinCols; ++c)
              h[((size_t)w * d.k + r) * kWinCols + c] = __float2half_rn((float)src(w, r, c));
        if (p->arena.alloc(&gdev, n * 2) || cudaMemcpy(gdev, h.data(), n * 2, cudaMemcpyHostToDevice))
          return fail(set_err(DPQ_ERR_CUDA, "G upload"));
      } else if (d.g_dtype == G_E4M3) {
        std::vector<unsigned char> h(n);
        for (int w = 0; w < L.n_win; ++w)
          for (int r = 0; r < d.k; ++r)
            for (int c = 0; c < kWinCols; ++c) {
              __nv_fp8_e4m3 v((float)(src(w, r, c) / rowscale[r]));
              h[((size_t)w * d.k + r) * kWinCols + c] = v.__x;
            }
        float* sdev = nullptr;
        if (p->arena.alloc(&gdev, n) || cudaMemcpy(gdev, h.data(), n, cudaMemcpyHostToDevice) ||
            p->arena.alloc_t(&sdev, d.k) ||
            cudaMemcpy(sdev, rowscale.data(), d.k * 4, cudaMemcpyHostToDevice))
          return fail(set_err(DPQ_ERR_CUDA, "G upload"));
        S.g_scale = sdev;
      } else {
        return fail(set_err(DPQ_ERR_ARG, "layer %d: unknown G dtype %d", i, d.g_dtype));
      }
      S.G = gdev;
    }
    p->gt_fb.push_back(0);
    if (S.sentinel == 0 && d.est_kind == EST_PROJECTION) {
      // fixed-point fraction bits of the engine's packed G.x words: a window
      // partial |G_k[w] . x[w]| <= maxl1 * 2^16 must stay below 2^46 (< the
      // 2^47 bias) after scaling by 2^fb (larger inputs raise the engine's
      // range flag, DPQ_ERR_RANGE)
      double maxl1 = 0.0;
      for (int r = 0; r < d.k; ++r) {
        double a = 0.0;
        for (int c = 0; c < L.cols; ++c) a += std::fabs(d.G[(size_t)r * L.cols + c]);
        maxl1 = std::max(maxl1, a);
      }
      int fb = 46 - (int)std::ceil(std::log2(std::max(maxl1, 1e-30) * 65536.0));
      p->gt_fb.back() = std::min(52, std::max(-16, fb));
      // tensor parallel shards of G (rows by k) must share the full layer's scale
      if (d.fx_bits_plus128 != 0) p->gt_fb.back() = d.fx_bits_plus128 - 128;
    }
    if (S.sentinel == 0 && d.prev_residual) p->any_prev = 1;
    p->sel.push_back(S);
    dpq_sel_desc hd = d;
    hd.G = nullptr;
    p->host.push_back(hd);
  }
  *out = p;
  return DPQ_OK;
}

extern "C" int dpq_plan_destroy(dpq_plan* p) {
  if (!p) return DPQ_OK;
  cudaSetDevice(p->store->device);
  cudaDeviceSynchronize();
  gemv_progs_release(p->gemv_progs);
  p->arena.release();
  delete p;
  return DPQ_OK;
}

extern "C" int dpq_select_gemv(dpq_plan* p, int layer, const float* x_dev, const float* est_in_dev,
                               float* y_dev, int32_t* bit_out_dev, float* est_out_dev,
                               float* exact_out_dev, void* stream) {
  if (!p || layer < 0 || layer >= (int)p->sel.size() || !x_dev || !y_dev)
    return set_err(DPQ_ERR_ARG, "dpq_select_gemv: bad arguments");
  dpq_store* s = p->store;
  CK(cudaSetDevice(s->device));
  cudaStream_t st = (cudaStream_t)stream;
  DevSel S = p->sel[layer];
  const bool exact_est = S.sentinel == 0 && S.est_kind == EST_EXACT;
  const bool want_exact = exact_out_dev != nullptr && S.l != S.h;
  if (!exact_est && !want_exact && (est_in_dev == nullptr || est_in_dev == x_dev)) {
    bool used = false;
    TRY(gv_run(s, p, layer, 0, x_dev, y_dev, bit_out_dev, est_out_dev, st, &used));
    if (used) return DPQ_OK;
    TRY(gemv_engine_run(s, p, layer, 0, x_dev, y_dev, bit_out_dev, est_out_dev, st, &used));
    if (used) return DPQ_OK;
  }
  reset_trace1<<<1, 32, 0, st>>>(s->tr_bits, s->tr_est, s->tr_exact);
  CK(cudaGetLastError());
  if (exact_est && est_in_dev) {
    // estimate = ||(W_h - W_l) x_in|| on the explicit estimator input first
    DevSel Se = S;
    OpDesc E = single_op(s, layer, Se, est_in_dev, s->est_buf);
    E.layer[0].dual = 1;
    E.n_trace = 1;
    E.main_decision = s->decision;
    E.layer[0].main_li = 0;
    TRY(run_op(E, s->ctl, s->n_sm, st, false));
    TRY(launch(decide_exact, dim3(1), dim3(256), 0, st, false, E, s->ctl));
    S.sentinel = 3;
  }
  OpDesc D = single_op(s, layer, S, x_dev, y_dev);
  D.est_in = exact_est ? nullptr : est_in_dev;
  D.layer[0].dual = (exact_est && !est_in_dev) || want_exact;
  TRY(run_op(D, s->ctl, s->n_sm, st, false));
  if (D.layer[0].dual) TRY(launch(finalize_dual, dim3(1), dim3(256), 0, st, false, D, s->ctl));
  copy_sel_outputs<<<1, 32, 0, st>>>(s->tr_bits, s->tr_est, s->tr_exact, bit_out_dev, est_out_dev,
                                     exact_out_dev);
  CK(cudaGetLastError());
  return DPQ_OK;
}

// ---------------------------------------------------------------------------
// standalone estimators
// ---------------------------------------------------------------------------
struct dpq_estimator {
  int device = 0;
  int kind = 0, k = 0, cols = 0;
  double slope = 0, intercept = 0;
  float* G = nullptr;      // [k][cols] fp32
  float* gx = nullptr;     // [k]
  double* sq = nullptr;    // [1]
  double* out = nullptr;   // [1]
  Arena arena;
};

namespace {
__global__ void est_rows_kernel(const float* __restrict__ G, int cols, const float* __restrict__ x,
                                float* __restrict__ gx) {
  __shared__ double red[32];
  const int r = blockIdx.x;
  double acc = 0.0;
  for (int c = threadIdx.x; c < cols; c += blockDim.x) acc += (double)G[(size_t)r * cols + c] * x[c];
  acc = block_sum_d(acc, red);
  if (threadIdx.x == 0) gx[r] = (float)acc;
}
__global__ void est_norm_kernel(const float* __restrict__ v, int n, int square_of_x, double slope,
                                double intercept, double* __restrict__ out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += (double)v[i] * v[i];
  acc = block_sum_d(acc, red);
  if (threadIdx.x == 0) out[0] = square_of_x ? slope * sqrt(acc) + intercept : sqrt(acc);
}
__global__ void sum_sq_tiles(const float* __restrict__ q, int n, double* __restrict__ out) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += (double)q[i];
  acc = block_sum_d(acc, red);
  if (threadIdx.x == 0) out[0] = sqrt(acc);
}
}  // namespace

extern "C" int dpq_estimator_create(int device, const dpq_sel_desc* sel, int cols, dpq_estimator** out) {
  if (!sel || !out || cols < 1 || (sel->est_kind != EST_LINEAR && sel->est_kind != EST_PROJECTION))
    return set_err(DPQ_ERR_ARG, "dpq_estimator_create: linear or projection estimator required");
  if (sel->est_kind == EST_PROJECTION && (sel->k < 1 || !sel->G))
    return set_err(DPQ_ERR_ARG, "dpq_estimator_create: projection needs G");
  CK(cudaSetDevice(device));
  dpq_estimator* e = new dpq_estimator();
  e->device = device;
  e->kind = sel->est_kind;
  e->k = sel->k;
  e->cols = cols;
  e->slope = sel->slope;
  e->intercept = sel->intercept;
  int r = e->arena.alloc_t(&e->out, 1);
  if (!r && e->kind == EST_PROJECTION) {
    std::vector<float> g((size_t)e->k * cols);
    for (size_t i = 0; i < g.size(); ++i) g[i] = (float)sel->G[i];
    r = e->arena.alloc_t(&e->G, g.size());
    if (!r) r = e->arena.alloc_t(&e->gx, e->k);
    if (!r && cudaMemcpy(e->G, g.data(), g.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
      r = set_err(DPQ_ERR_CUDA, "G upload");
  }
  if (r) {
    e->arena.release();
    delete e;
    return r;
  }
  *out = e;
  return DPQ_OK;
}

extern "C" int dpq_estimator_eval(dpq_estimator* e, const float* x_dev, double* est_out_host, void* stream) {
  if (!e || !x_dev || !est_out_host) return set_err(DPQ_ERR_ARG, "dpq_estimator_eval: bad arguments");
  CK(cudaSetDevice(e->device));
  cudaStream_t st = (cudaStream_t)stream;
  if (e->kind == EST_PROJECTION) {
    est_rows_kernel<<<e->k, 256, 0, st>>>(e->G, e->cols, x_dev, e->gx);
    est_norm_kernel<<<1, 256, 0, st>>>(e->gx, e->k, 0, 0.0, 0.0, e->out);
  } else {
    est_norm_kernel<<<1, 256, 0, st>>>(x_dev, e->cols, 1, e->slope, e->intercept, e->out);
  }
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(est_out_host, e->out, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return DPQ_OK;
}

extern "C" int dpq_estimator_destroy(dpq_estimator* e) {
  if (!e) return DPQ_OK;
  cudaSetDevice(e->device);
  cudaDeviceSynchronize();
  e->arena.release();
  delete e;
  return DPQ_OK;
}

extern "C" int dpq_exact_error(dpq_store* s, int layer, int l, int h, const float* x_dev, double* out_host,
                               void* stream) {
  if (!s || layer < 0 || layer >= (int)s->layers.size() || !x_dev || !out_host)
    return set_err(DPQ_ERR_ARG, "dpq_exact_error: bad arguments");
  const DevLayer& L = s->layers[layer];
  if (l >= h) return set_err(DPQ_ERR_ARG, "need l < h, got (%d, %d)", l, h);
  if (l < L.b_min || h > L.n_bits) return set_err(DPQ_ERR_ARG, "bitwidth outside [%d, %d]", L.b_min, L.n_bits);
  CK(cudaSetDevice(s->device));
  cudaStream_t st = (cudaStream_t)stream;
  DevSel S{};
  S.l = l;
  S.h = h;
  S.prefill_bit = h;
  S.sentinel = 1;
  S.T = INFINITY;
  OpDesc D = single_op(s, layer, S, x_dev, s->est_buf);
  D.layer[0].dual = 1;
  D.layer[0].trace_idx = -1;
  D.n_trace = 0;
  TRY(run_op(D, s->ctl, s->n_sm, st, false));
  double* dout = reinterpret_cast<double*>(s->tr_est);   // 4 floats of scratch = 2 doubles
  sum_sq_tiles<<<1, 256, 0, st>>>(D.dual_sq, L.n_tiles, dout);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out_host, dout, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return DPQ_OK;
}

#include "dpq_session.inc"
