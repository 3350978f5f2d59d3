// plan.hpp - host-side planner for the B200 tcFFT passes (no CUDA dependency).
//
// A plan is a list of passes; a pass is one persistent kernel launch that
// reads every element once from HBM and writes it once.  Inside a pass each
// CTA loops over "chunks" of E complex elements (several short transforms or a
// strip of columns), runs S DFT-as-GEMM stages on the tensor cores and stores
// the chunk back.  All index math (which butterfly a TMEM lane owns at each
// stage, where its outputs go, which twiddle they need) is resolved here, on
// the host, into small per-(stage, tile, lane) tables, so the kernel only does
// affine address arithmetic.  See DESIGN.md for the dataflow.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace tcfft {

constexpr int kMaxStages = 3;
constexpr int kLanes = 128;  // M of every tcgen05.mma tile
constexpr int kMaxLog2_1D = 30;  // 1D N <= 2^30 (three-step, N1 N2 N3 with N3 <= 256)

enum PassKind : int32_t {
  kPassRow = 0,    // contiguous transforms: element n of transform tr at tr*N + n
  kPassStrip = 1,  // column strip: element n of column tr at n*C + tr (2D column / four-step pass 1)
  kPassRowT = 2,   // contiguous rows in, transposed columns out (four-step pass 2)
  kPassStripT = 3, // column strip in, each column written as a contiguous row (three-step pass A)
  kPassRowTB = 4,  // rows of a blocked [block][row][Bw] array in, transposed columns out (two-pass pass 2)
};

enum IoMode : int32_t {
  kIoBox = 0,    // 3D tensor map {C, rows, 1} over images x rows x cols
  kIoFlat = 1,   // 2D tensor map [total/W][W] over a contiguous chunk
  kIoRank1 = 2,  // 1D tensor map [total] in 256-element boxes
  kIoPitch = 3,  // per-transform 1D bulk copies into a padded staging pitch
  kIoBoxR = 4,   // 4D tensor map {C, 256, rows/256, 1}: a > 256-row strip in ONE box
  kIoFlat3 = 5,  // 3D tensor map {W, 256, n_sub} over [total/W/256][256][W]: one box per chunk
  kIoBlk = 6,    // 4D tensor map {C*W, 1, blocks, 1} over [images][blocks][rows/C][C*W]: C rows of every block
  kIoLinear = 7, // the whole staging tile, byte for byte, to/from chunk * E (one non-tensor bulk copy)
  kIoPeer = 8,   // the staging tile in `npeer` row slices, slice h byte for byte to peer h's buffer (distributed plans)
};

// How one side (load or store) of a pass moves a chunk between HBM and SMEM.
struct IoDesc {
  int32_t mode = kIoFlat;
  int32_t W = 0, swz = 0;
  int32_t box_rows = 0, n_sub = 0, sub_bytes = 0, chunk_rows = 0;
  int32_t C = 0, spi = 0;  // box: columns per chunk, chunks per image
  int64_t images = 0;
  int32_t rows = 0, cols = 0;
  int64_t total = 0;
  // box mode, optional explicit strides (elements; 0 = dense images x rows x cols)
  // and a split image index img = outer * img_split + inner (4D tensor map:
  // inner stride img_stride, outer stride img_stride2)
  int64_t row_stride = 0, img_stride = 0, img_stride2 = 0;
  int32_t img_split = 0;
  int32_t npeer = 0;        // kIoPeer: slices (ranks); slice bytes = sub_bytes
  int64_t peer_blk0 = 0;    // kIoPeer: global column block of chunk 0
};

struct StageInfo {
  int32_t R;        // radix
  int32_t n2;       // product of earlier radices (reference kernels.py:323 "n2")
  int32_t KP, NP;   // MMA K and N (2R padded up to 16)
  int32_t tiles;    // E / (128 R)
  int32_t sbo;      // A operand stride between 8-row core-matrix groups (bytes), SS stages
  int32_t tile_bytes;  // A operand bytes per 128-row tile
  int32_t b_off;    // byte offset of this stage's B matrix in the B blob
  int32_t b_bytes;
  int32_t t_off;    // byte offset of the writer twiddle table (float4 [R'][R/2]); -1 if final
  int32_t hstep;    // writer: byte step between successive 8-output chunks
  int32_t im_off;   // writer: byte offset of the imaginary plane (R' * 16)
};

// Per (stage, tile, lane) row record, 32 bytes, read once per CTA.
struct RowInfo {
  int32_t gbase;  // stage 1: word address (staging) of input m = 0
  int32_t addr;   // writer: byte offset of its first 16B chunk in the next A tile;
                  // final stage: word address (staging) of output j = 0
  int32_t mp;     // writer: next-stage input index m'
  int32_t tw;     // 1 if the writer's c differs from 1 (stage >= 2)
  float cr, ci;   // writer: twiddle of output j = 0, c = W_{R' n2'}^{m' k}
  float wr, wi;   // writer: per-output ratio w = W_{R R'}^{m'}; output j gets c * w^j
};

struct PassPlan {
  int32_t kind;     // PassKind
  int32_t N;        // transform length of this pass
  int32_t E;        // complex elements per chunk
  int32_t T;        // transforms per chunk
  int32_t S;        // stages
  StageInfo st[kMaxStages];
  int32_t gstride;  // staging words between successive gather inputs m
  int32_t ostride;  // staging words between successive final outputs j
  int32_t swz_in, swz_out;  // 128B/64B/32B swizzle masks (0x70/0x30/0x10) or 0
  int64_t count;    // transforms in the pass (row) or columns (strip)
  int64_t chunks;
  // strip geometry (kind == kPassStrip): images x rows(=N) x cols, C columns
  // of IMG images per chunk
  int64_t images;
  int32_t rows, cols, C, IMG;
  // TMA: flat contiguous chunk ([total/W][W] view) or 3D column box
  int32_t flat, W, box_rows, n_sub, sub_bytes;
  int32_t pitch_mode, pitch;  // row inputs, 64 <= N <= 1024: padded per-transform staging (words)
  IoDesc in, out;
  int64_t tw4_total;   // four-step pass 1: N of the full transform (extra twiddle), else 0
  int32_t tw4_shift;   // twiddle exponent uses (column >> tw4_shift) (three-step pass B), else 0
  int64_t tw4_col0 = 0;  // global column of the pass's first column (distributed plans), added to the twiddle base
  int32_t ws_in, ws_out;  // pass reads / writes the plan workspace
  int32_t smem_tw4;
  int64_t total;
  // shared-memory carve-up (bytes, relative to the 1024-aligned base)
  int32_t smem_in, smem_a, smem_b, smem_t, smem_bar, smem_bytes;
  int32_t a_bytes;   // A buffer size (>= E*4, also used as output staging)
  int32_t tmem_cols; // allocation (power of two >= 32)
  int32_t tmem_a_cols;
  int32_t ctas_per_sm;
  int32_t planar0 = 0;       // stage-1 A operand in planar K order (radix-64 first stage)
  int32_t nwg = 1;           // warpgroups per CTA (2 for one-CTA-per-SM passes with even tile counts)
  int32_t a_bufs;            // 1 or 2 A / output-staging buffers
  int32_t onebuf = 0;        // single-buffer pass (kernel ONEBUF): staging == A buffer, 2 CTAs/SM at E = 16384
  int32_t tmem_cols_needed;
  std::vector<RowInfo> rows_tab;   // [S][tiles_max][128]
  int32_t tiles_max;
  std::vector<uint16_t> bblob;     // fp16 B matrices, UMMA K-major core-matrix order
  std::vector<float> tblob;        // writer twiddle tables, 8 floats per (m', j-pair)
};

struct Plan {
  int32_t dims = 1;
  int32_t nx = 0, ny = 0;
  int64_t batch = 0;
  size_t ws_bytes = 0;
  int32_t dist = 0;         // distributed single-transform plan: 1 NCCL-exchange variant, 2 fused (peer stores)
  int64_t groups = 1;       // passes run once per group of transforms
  size_t group_bytes = 0;   // input / output bytes of one group
  std::vector<PassPlan> passes;
};

// Experiment hooks (A/B measurements only, never needed by users): returns
// getenv(name) when the process sets TCFFT_EXPERIMENTS=1, else nullptr, so a
// stray environment variable cannot change a plan.  The only getenv calls in
// the library are inside this gate.
const char* experiment_env(const char* name);

// Radix list chosen for a single-pass transform of length n (product == n).
std::vector<int> choose_radices(int n, int kind = kPassRow, bool twiddled = false);
// row-block interleave of a writer stage of radix R (kernel Cfg::HSTEP mirrors it)
int writer_groups(int R, int rows_next);
int chunk_elems_for(int n);
int pitch_pad_words(int n);

// Builds a pass.  kind/geometry as in PassPlan; returns false on unsupported size.
// blk: block width Bw of a kPassRowTB input; want_E: chunk size override (0 = default)
bool build_pass(PassPlan& p, int kind, int N, int64_t count, int64_t images, int cols, std::string* err,
                int64_t tw4_total = 0, int tw4_shift = 0, int blk = 0, int want_E = 0);
// Builds the whole plan (host-only, no CUDA calls).
int build_plan(Plan& plan, int dims, int nx, int ny, int64_t batch, std::string* err);
// Distributed single transform (rank `rank` of `world`): the two local passes
// of a four-step N = N1 N2 split by columns (pass 0) and by rows (pass 1); the
// caller exchanges the data between them (paper_2104_11471_b200/dist.py).
// fused: pass 0 stores each N1/world-row slice of its staging tile straight
// into the owning rank's receive buffer (peer memory, kIoPeer) in the blocked
// layout [N2/C][N1/world][C], pass 1 is the blocked-rows pass (no exchange
// collective, no unpack).
int build_plan_dist(Plan& plan, int nx, int rank, int world, std::string* err, bool fused = false);

}  // namespace tcfft
