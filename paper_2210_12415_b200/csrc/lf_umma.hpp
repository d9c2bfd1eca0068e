// lf_umma.hpp — planning and launch of the tcgen05 (UMMA) contraction
// kernel that runs GMM (K3) and C2D (K4) directly on tuned layouts.
//
// One generic warp-specialised kernel serves both operators. Everything
// layout-specific is resolved on the host into tables:
//   * per CTA tile: TMA box coordinates of the A/B operands (tile part),
//     the output base offset, valid rows/cols and the logical N base (bias);
//   * per K stage: TMA coordinate increments (stage part);
//   * per tile row / column: physical output offsets.
// A coordinate of any operand dim is tile_part + stage_part because every
// physical digit of a template layout belongs to exactly one logical dim
// (space.cpp:174-417), and the unfolded input offset digit is V*h1 + rh.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "lf_core.hpp"

namespace lfg {

struct PairPlan;    // lf_pair.hpp
struct PairLaunch;

enum { UMMA_GEMM = 0, UMMA_CONV = 1 };
enum { EPI_NONE = 0, EPI_BIAS = 1, EPI_RELU = 2, EPI_RESIDUAL = 3, EPI_GELU = 4 };
#ifdef __CUDACC__
// GELU as lfgpu.h defines it (exact erf form), in fp32 in the epilogue.
__device__ __forceinline__ float epi_gelu(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }
#endif
constexpr int kMaxEpi = 4;
constexpr int kMaxBoxes = 4;
constexpr int kMaxTaps = 32;  // taps of the halo C2D path (KH*KW)
// Epilogue transpose buffers: 8 warps x 32 rows x 36 floats (k_umma.cu).
constexpr int kEpiSmemBytes = 8 * 32 * 36 * 4;

struct EpiOp {
  int32_t kind = EPI_NONE;
  int32_t tensor = -1;      // plan tensor index of the bias / residual operand
  int32_t out_tensor = -1;  // node output this op produces (chain bookkeeping)
  const float* ptr = nullptr;
};

// Host description of one operand's TMA view and UMMA SMEM descriptor.
struct OperandView {
  int32_t rank = 0;
  int32_t elem_bytes = 2;  // 2: bf16, 4: fp32 (output views)
  uint64_t dims[5] = {};
  uint64_t strides[5] = {};  // bytes, dims 1..rank-1
  uint32_t box[5] = {};
  uint32_t estride[5] = {1, 1, 1, 1, 1};
  int32_t swizzle = 128;  // bytes: 32 / 64 / 128
  int32_t mn_major = 0;
  int32_t boxes = 1;      // TMA loads per stage
  int32_t box_bytes = 0;  // bytes one load writes
  int32_t slot_bytes = 0; // SMEM bytes reserved per box (>= box_bytes, aligned)
  uint32_t sbo = 0, lbo = 0;
  uint32_t k_adv = 0;     // descriptor start-address advance per UMMA K=16 step
};

// A Padding absorbed into the producing C2D's epilogue (the producer writes
// the consumer's padded, possibly unfolded layout directly; PAPER.md:379-381,
// lower.cpp:228-238). Output element (n, c, h, w) lands at every physical
// position of the bf16 destination whose logical coordinate is
// (n, c, h+pad, w+pad): per unfolded dim the tiles t with
// t*S <= x < t*S + B (exact tilings only), offset
// n*sN + (c/ic)*sC0 + (c%ic)*sC1 + t_h*sHt + (x_h - t_h*S_h)*sHo + (same for W).
// The pad ring is zeroed once at plan build and never written.
struct ScatterDesc {
  int32_t enabled = 0;
  int32_t pad = 0;
  int32_t ic = 1;           // channel brick (c % ic inner)
  int32_t Th = 1, Bh = 1, Sh = 1 << 30, Tw = 1, Bw = 1, Sw = 1 << 30;
  int64_t sN = 0, sC0 = 0, sC1 = 0, sHt = 0, sHo = 0, sWt = 0, sWo = 0;
  void* dst = nullptr;      // bf16 buffer of the padded tensor
};

// Descriptor of a Padding(pad) output layout for the epilogue scatter; false
// when the layout is not a separable (N, C, H, W) brick form.
bool umma_scatter_desc(const std::vector<Dim>& xp_log, const Seq& xp_seq, int64_t pad,
                       ScatterDesc* sd, std::string* why);

struct TileEntry {  // 192 bytes
  int32_t ca[kMaxBoxes][5];
  int32_t cb[kMaxBoxes][5];
  int64_t out_base;
  int32_t rows, cols;
  int32_t n_base;
  int32_t org[3];  // C2D: logical (n, h, w) of the tile origin (epilogue scatter)
};

struct StageEntry {  // 40 bytes
  int32_t sa[5];
  int32_t sb[5];
};

// TMA-store epilogue (store mode 2): the fp32 output tile is staged in SMEM
// (16 columns = 64 bytes per row, SWIZZLE_64B) and written by
// cp.async.bulk.tensor; `row_pos[r]` is accumulator row r's row in the box
// (-1: not an output row), `tile_coords` the box origin of every tile.
struct OutStore {
  bool ok = false;
  OperandView O;                     // fp32 view of the output (box: 16 cols x tile rows)
  int col_dim = 0;                   // view dim of the columns (0 unless transposed)
  int col_stride = 0;                // transposed box: element stride of one column plane
  std::vector<int32_t> tile_coords;  // ntiles x 5
  std::vector<int32_t> row_pos;      // 128
  int box_rows = 0;                  // rows of one staged chunk
  std::string why;
};

struct UmmaPlan {
  int kind = UMMA_GEMM;
  int BM = 128, BN = 128;
  int KC = 64;          // K elements per stage
  int pipe = 4;         // SMEM pipeline depth
  int persistent = 0;
  int split_pref = 0;   // schedule `order`: 0 heuristic split-K, 1 never, 2 at least 2
  // Halo C2D: per K stage, `ntaps` UMMA groups; tap t reads A at +a_tap[t]
  // bytes and B at +t*b_tap bytes inside the stage (ntaps = 1: plain GEMM).
  int ntaps = 1;
  std::vector<int32_t> a_tap{0};
  int b_tap = 0;
  std::vector<int32_t> b_tapv;  // per-tap B offsets (empty: t * b_tap)
  int trans = 0;                // C2D with output channels as UMMA rows (pixels as N)
  int swap_ab = 0;              // A views the node's second operand (weights), B the first
  int wres = 0;          // halo C2D: weights resident in SMEM (one output-channel tile)
  OutStore ost;          // TMA-store epilogue, when the output tile is a TMA box
  int tma_store = 0;     // schedule `vectorize`: use the TMA-store epilogue when legal
  std::vector<int32_t> row_rel;  // C2D: (dh << 16) | dw of accumulator row r from the tile origin
  ScatterDesc scatter;   // Padding absorbed into this epilogue (runtime fills it)
  OperandView A, B;
  std::vector<TileEntry> tiles;
  std::vector<StageEntry> stages;
  std::vector<int64_t> row_off, col_off;
  EpiOp epi[kMaxEpi];
  int epi_count = 0;
  const void* a = nullptr;
  const void* b = nullptr;
  float* out = nullptr;
  void* out_bf16 = nullptr;  // optional bf16 copy written by the epilogue
  int out_stream = 0;        // output is a graph output nothing reads back: streaming (evict-first) stores
  std::string summary;
  // GEMM on the CTA-pair kernel (k_pair.cu) when its tile is legal: the
  // fields above except epi/a/b/out are then unused.
  std::shared_ptr<PairPlan> pair;
};

// Per-launch device state (tables uploaded, tensor maps encoded).
struct UmmaLaunch {
  CUtensorMap tma_a, tma_b;
  int chain_slot = -1;  // diagnostics: this launch's slot in the chain trace (plan step index)
  void* d_tiles = nullptr;
  void* d_stages = nullptr;
  void* d_rows = nullptr;
  void* d_cols = nullptr;
  int ntiles = 0, nstages = 0, BN = 0, KC = 0, pipe = 0, tmem_cols = 0, nprod = 1;
  int a_boxes = 0, b_boxes = 0, a_slot = 0, b_slot = 0, a_bytes = 0, b_bytes = 0;
  uint64_t a_desc = 0, b_desc = 0;  // descriptor templates (start address filled on device)
  uint32_t a_kadv = 0, b_kadv = 0;
  uint32_t idesc = 0;
  int epi_kinds[kMaxEpi] = {};
  const float* epi_ptr[kMaxEpi] = {};
  int epi_count = 0;
  float* out = nullptr;
  void* out_bf16 = nullptr;
  int out_stream = 0;
  size_t smem = 0;
  int grid = 0;
  int per_sm = 1;  // CTAs that fit on one SM (SMEM / TMEM)
  int ring_bytes = 0;
  int table_ints = 0;            // [stages | col_off | row_off] int32 count
  int ntaps = 1, b_tap = 0, bias_rows = 0;
  int32_t b_tapv[kMaxTaps] = {};
  int wres = 0, w_chunk = 0, w_tx = 0;
  CUtensorMap tma_o, tma_ob;     // store mode 2: fp32 output and its bf16 copy
  int stg_off = 0, stg_f32 = 0, stg_bf = 0;
  int stg_nbuf = 1, epi_region = kEpiSmemBytes;
  int epi_alias = 0;  // epilogue buffers alias the operand ring (<= 1 unit per CTA)
  int stg_cstride = 0, stg_cdim = 0;  // transposed TMA-store box (OutStore::col_stride / col_dim)
  void* d_tcoords = nullptr;
  ScatterDesc scatter;
  int red_bytes = 0;
  int32_t a_tap[kMaxTaps] = {};
  int store_mode = 0;           // 1: transposed float4 row stores; 0: generic
  int64_t col0 = 0;
  int splits = 1;               // split-K factor (k_umma.cu)
  int dual = 0;                 // two MMA issuers (warps 1 and 3) on alternate units
  int blocked = 0;              // contiguous unit chunks per CTA (loop point parallel = 1)
  int xsplit = 0;               // split-K over DSMEM inside a cluster (one unit per CTA)
  int w_prewait = 0;            // set by the plan: resident weights loaded before the PDL wait
  float* ws = nullptr;          // split-K partial tiles
  int* counters = nullptr;      // split-K per-tile arrival counters
  std::shared_ptr<void> owner;  // keeps the device tables alive
  std::shared_ptr<PairLaunch> pair;  // launch through k_pair.cu instead
};

bool umma_plan_gemm(const std::vector<Dim>& a_log, const Seq& a_seq, const std::vector<Dim>& b_log,
                    const Seq& b_seq, const std::vector<Dim>& c_log, const Seq& c_seq,
                    const lfgpu_sched& s, UmmaPlan* out, std::string* why, int rows_per_tile = 128);
bool umma_plan_conv(const std::vector<Dim>& x_log, const Seq& x_seq, const std::vector<Dim>& k_log,
                    const Seq& k_seq, const std::vector<Dim>& y_log, const Seq& y_seq,
                    int64_t stride, const lfgpu_sched& s, UmmaPlan* out, std::string* why);
// Tensor map of an operand view at `base`, its UMMA SMEM descriptor bits
// (start address added on the device) and the kind::f16 instruction
// descriptor (shared with the CTA-pair kernel, k_pair.cu).
CUtensorMap umma_encode(const OperandView& v, const void* base);
uint64_t umma_desc_bits(const OperandView& v);
uint32_t umma_idesc(int M, int N, bool a_mn, bool b_mn);
int umma_num_sms();
// True when TMA can encode the view (checked with a dummy base address).
bool umma_view_encodable(const OperandView& v, std::string* why);
// Encodes tensor maps and uploads tables (needs a, b, out set).
UmmaLaunch umma_prepare(const UmmaPlan& p);
cudaError_t umma_launch(const UmmaLaunch& L, cudaStream_t stream);
// Debug: when set, every umma launch writes 8 %globaltimer checkpoints per CTA.
void* umma_debug_buffer();
void umma_set_debug_buffer(void* p);

}  // namespace lfg
