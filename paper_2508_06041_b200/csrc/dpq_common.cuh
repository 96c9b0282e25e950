// Shared device/host structures for the DP-LLM decode hot path on sm_100a.
//
// Device layout of one quantized layer (rows x cols, n_bits nested planes):
//   plane p (0 = MSB; the b-bit code is planes 0..b-1, reference quant.py:74)
//   is stored window-major: [p][window w][row tile rt][chunk c][lane l][16 B]
//   window = 512 input columns, row tile = 32 output rows, lane l = row % 32.
//   Lane l's 64-byte segment holds one byte per "step" s = 16c + byte-in-chunk;
//   step s covers column group g = (l + s) mod 64 (8 columns 512w+8g..+7, bit t
//   of the byte = column 8g+t), stored as (e - [l+s >= 64]) mod 256. That
//   rotation makes the byte-LUT lookups of the 32 lanes hit 32 distinct banks
//   and lets one PRMT form the shared-memory address (see lut_lookup()).
//
// Byte LUT of a window (shared memory, 257 rows x 64 slots x fp32):
//   row e, slot g = sum_{t: bit t of e} x[512w + 8g + t]; row 256 = 0.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dpq {

constexpr int kWinCols = 512;          // columns per window
constexpr int kGroups = 64;            // 8-column groups per window
constexpr int kTileRows = 32;          // rows per tile (one per lane)
constexpr int kTileBytes = 2048;       // bytes of one (plane, window, tile)
constexpr int kLutRows = 257;
constexpr int kLutBytes = kLutRows * kGroups * 4;   // 65792
constexpr int kMaxOpLayers = 3;
constexpr int kThreads = 512;          // op kernel block size
constexpr int kMaxK = 128;             // max projection rank

enum GDtype : int { G_F32 = 0, G_F16 = 1, G_E4M3 = 2 };
enum EstKind : int { EST_NONE = 0, EST_LINEAR = 1, EST_PROJECTION = 2, EST_EXACT = 3 };
enum InMode : int { IN_IDENT = 0, IN_RMS = 1, IN_SILU = 2 };
enum OutMode : int { OUT_STORE = 0, OUT_ADD = 1 };
enum StepMode : int { MODE_PREFILL = 0, MODE_DYNAMIC = 1 };

// Immutable, device-resident layer of the store.
struct DevLayer {
  const uint4* planes;      // plane p at planes + p * plane_stride16
  const float* lo;          // [rows_pad]
  const float* span;        // [rows_pad] (hi - lo)
  long long plane_stride16; // uint4 per plane = n_win * n_tiles * 128
  int rows, cols, n_bits, b_min, n_win, n_tiles;
};

// Selector parameters of one layer (from the plan), device copy.
struct DevSel {
  int l, h, prefill_bit;
  int sentinel;             // 0 = estimate, 1 = T=+inf (low), 2 = T=-inf (high)
  int est_kind;             // EstKind
  int k, g_dtype;
  int prev_residual;        // estimator input_source == previous_residual
  double T, slope, intercept;
  const void* G;            // [n_win][k][512] of g_dtype
  const float* g_scale;     // [k] per-row scale (e4m3) or nullptr
};

// Per-session mutable control block (device memory, read by every kernel).
struct Control {
  int mode;                 // StepMode                      (host-written)
  int token;                // token being processed          (host or argmax)
  int force;                // decisions replaced by forced_bits (host-written)
  int pos;                  // position of the token being processed
  int trace_step;           // index of the next dynamic trace record
  int snap_w, snap_r;       // snapshot slots written / read as "previous step"
  int has_prev;             // a previous-step snapshot exists
  int prime;                // prime_from_prefill
  int async_prev_block;     // async_rule == "prev_block"
  int n_steps_done;
  const signed char* forced_bits;   // [n_trace_layers] (when force)
};

struct OpSync {
  unsigned arrive;
  unsigned gen;
  unsigned pad[30];         // keep each sync object on its own 128 B line
};

// One layer inside an op (op = layers sharing one input vector).
struct OpLayer {
  DevLayer L;
  DevSel S;
  int out_off;              // first output row inside the op output
  int tile_off;             // first tile inside the op (counters / partials)
  int trace_idx;            // layer index in the trace, -1 = untraced
  int dual;                 // also produce y at l and h (exact / track_exact)
  int snap_in;              // snapshot index of this op's input one block earlier
  int main_li;              // estimation ops: index of the layer in the main op
};

struct OpDesc {
  int n_layers;
  int cols, n_win, total_tiles, rows_total_pad;
  int in_mode;              // InMode
  int out_mode;             // OutMode
  int need_snap;            // write the raw input + stats into snapshots
  int snap_idx;             // this op's input snapshot index
  float eps;
  const float* in0;         // input (IN_SILU: up half)
  const float* in1;         // IN_SILU: gate half
  float* out;               // [rows_total] (OUT_ADD: residual, updated in place)
  float* out_lo;            // dual: y at l  [rows_total]
  float* out_hi;            // dual: y at h  [rows_total]
  float* dual_sq;           // dual: per layer sum (y_h - y_l)^2, [n_layers]
  // scratch
  float* part;              // [n_win][rows_total_pad]
  float* part_lo;           // dual: S at l planes [n_win][rows_total_pad]
  float* gx_part;           // [n_layers][n_win][kMaxK]
  double* win_stats;        // [n_win][4] = (sum x, sum x^2, sum xp^2, -)
  float* op_stats;          // [4] = (sum x, sum x^2, inv, -) of this op's input
  unsigned* tile_cnt;       // [total_tiles]
  int* decision;            // [n_layers] selected bits (this step)
  int* main_decision;       // estimation ops: the main op's decision array
  const float* est_in;      // standalone select_gemv: explicit estimator input
  OpSync* sync;
  unsigned* ctr;            // per-op counters [128]: gdone, opdone, warr[n_win], tgrab[n_win]
  long long* gxa;           // per-op projection accumulators [kMaxOpLayers][kMaxK], fixed point 2^-40
  // snapshots (async estimator inputs), each [2 slots][n_snap][snap_stride]
  float* snap;              // raw inputs
  float* snap_stats;        // [2][n_snap][4] = (sum, sumsq, inv, -)
  int snap_stride;
  int n_snap;
  // trace
  signed char* tr_bits;     // [max_steps][n_trace]
  float* tr_est;            // [max_steps][n_trace]
  float* tr_exact;          // [max_steps][n_trace]
  int n_trace;
  int max_steps;
  unsigned long long* dbg;  // optional per-CTA phase timestamps [grid][8] (globaltimer ns)
  OpLayer layer[kMaxOpLayers];
};

}  // namespace dpq
