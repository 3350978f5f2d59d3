// tcfft_api.cu - C ABI (include/tcfft_b200.h): plan objects, device tables,
// TMA tensor maps and kernel dispatch for the sm_100a FFT passes.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tcfft_b200.h"
#include "fft_kernel.cuh"
#include "plan.hpp"

using tcfft::KParams;
using tcfft::PassPlan;

namespace {

using KernelFn = void (*)(CUtensorMap, CUtensorMap, KParams);

struct KernelEntry {
  int E, R1, R2, R3, mode, tw4, nwg, onebuf;
  const void* fn;
  void (*launch)(dim3, int, cudaStream_t, const CUtensorMap&, const CUtensorMap&, const KParams&);
};

// Programmatic dependent launch (default on, TCFFT_PDL=0 disables): a pass
// kernel may start launching while the previous kernel on the stream retires;
// its CTAs stage their constants and wait (griddepcontrol.wait) before the
// first TMA touches the data, so stream order is preserved.
static int pdl_mode() {
  static const int m = [] {
    const char* e = tcfft::experiment_env("TCFFT_PDL");
    return e ? std::atoi(e) : 1;
  }();
  return m;
}

template <int E, int R1, int R2, int R3, int MINB, int MODE, bool TW4, int NWG, bool OB>
void launch_tpl(dim3 grid, int smem, cudaStream_t st, const CUtensorMap& a, const CUtensorMap& b,
                const KParams& p) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(128 * NWG);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = p.pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, tcfft::fft_pass_kernel<E, R1, R2, R3, MINB, MODE, TW4, NWG, OB>, a, b, p);
}

#define KENTRYX(E, R1, R2, R3, MB, MODE, TW, NWG, OB)                                                   \
  {                                                                                                     \
    E, R1, R2, R3, MODE, TW, NWG, OB, (const void*)&tcfft::fft_pass_kernel<E, R1, R2, R3, MB, MODE, TW, NWG, OB>, \
        &launch_tpl<E, R1, R2, R3, MB, MODE, TW, NWG, OB>                                               \
  }
#define KENTRYW(E, R1, R2, R3, MB, MODE, TW, NWG) KENTRYX(E, R1, R2, R3, MB, MODE, TW, NWG, false)
#define KENTRY(E, R1, R2, R3, MB, MODE, TW) KENTRYW(E, R1, R2, R3, MB, MODE, TW, 1)
// single-buffer passes, two CTAs per SM (plan.cpp PassPlan::onebuf)
#define KONE(E, R1, R2, R3, MODE, TW) KENTRYX(E, R1, R2, R3, 2, MODE, TW, 1, true)
#define KROW(E, R1, R2, R3, MB) KENTRY(E, R1, R2, R3, MB, 0, false)
#define KSTRIP(E, R1, R2, R3, MB) KENTRY(E, R1, R2, R3, MB, 1, false)
#define KBOTH(E, R1, R2, R3, MB) KROW(E, R1, R2, R3, MB), KSTRIP(E, R1, R2, R3, MB)
#define KFOUR(E, R1, R2, R3, MB) KENTRY(E, R1, R2, R3, MB, 1, true), KENTRY(E, R1, R2, R3, MB, 2, false)

// Every (chunk size, radix list, mode) the planner can emit: contiguous row
// passes, column-strip passes (2D), and the two four-step passes (strip +
// twiddle, rows in / transposed out) for 1D sizes 2^15 .. 2^24.
const KernelEntry kKernels[] = {
    KBOTH(1024, 2, 0, 0, 4),      KBOTH(2048, 4, 0, 0, 4),      KBOTH(4096, 8, 0, 0, 4),
    KBOTH(4096, 16, 0, 0, 4),     KBOTH(4096, 32, 0, 0, 4),     KBOTH(4096, 8, 8, 0, 4),
    KBOTH(4096, 16, 8, 0, 4),     KBOTH(4096, 16, 16, 0, 4),    KBOTH(4096, 16, 32, 0, 4),
    KBOTH(4096, 32, 32, 0, 4),    KBOTH(4096, 16, 16, 8, 4),    KBOTH(4096, 16, 16, 16, 4),
    KROW(8192, 16, 16, 32, 2),    KSTRIP(8192, 16, 16, 8, 2),   KROW(16384, 16, 32, 32, 1),
    KROW(8192, 16, 16, 16, 2),    KROW(8192, 16, 32, 0, 2),     KROW(8192, 16, 16, 0, 2),
    KSTRIP(16384, 16, 16, 16, 1),
    // four-step: N1 / N2 in {128 .. 4096}
    KFOUR(4096, 16, 8, 0, 4),     KFOUR(4096, 16, 16, 0, 4),    KFOUR(4096, 16, 32, 0, 4),
    KFOUR(4096, 32, 32, 0, 4),    KFOUR(8192, 16, 16, 8, 2),    KFOUR(16384, 16, 16, 16, 1),
    KFOUR(16384, 16, 16, 8, 1),
    // strided passes of 2048 / 4096 with a radix-64 first stage (plan.cpp choose_radices)
    KSTRIP(8192, 64, 32, 0, 2),   KSTRIP(16384, 64, 64, 0, 1),  KFOUR(8192, 64, 32, 0, 2),
    KFOUR(16384, 64, 64, 0, 1),
    // three-step passes A / B (strip + twiddle) of length 64, pass C (strips in,
    // 4D natural-order store out) of length 64 .. 256
    KENTRY(4096, 8, 8, 0, 4, 1, true),  KENTRY(4096, 8, 16, 0, 4, 1, true), KENTRY(4096, 8, 16, 0, 4, 3, false),
    KSTRIP(4096, 8, 16, 0, 4),    KENTRY(4096, 8, 16, 0, 4, 2, false),  KENTRY(4096, 8, 8, 0, 4, 3, false), KENTRY(4096, 16, 8, 0, 4, 3, false),
    KENTRY(4096, 16, 16, 0, 4, 3, false),
    // wider 2D column strips (plan.cpp build_pass; 256: TCFFT_SCHUNK_256 experiment)
    KSTRIP(8192, 16, 32, 0, 2),   KSTRIP(8192, 32, 32, 0, 2),   KSTRIP(16384, 64, 32, 0, 1),
    KSTRIP(8192, 16, 16, 0, 2),   KSTRIP(8192, 8, 64, 0, 2),    KSTRIP(8192, 16, 64, 0, 2),
    KROW(8192, 64, 64, 0, 2),
    // one-CTA-per-SM passes with two warpgroups (plan.cpp PassPlan::nwg)
    KENTRYW(16384, 16, 32, 32, 1, 0, false, 2), KENTRYW(16384, 64, 64, 0, 1, 1, false, 2),
    KENTRYW(16384, 64, 32, 0, 1, 1, false, 2),
    // single-buffer 16384-element chunks (two CTAs per SM): 1D 16384 rows, 2D
    // 2048 / 4096 column strips, two-pass 2^22 (strip + twiddle, transposed rows)
    KONE(16384, 16, 32, 32, 0, false), KONE(16384, 64, 32, 0, 1, false), KONE(16384, 64, 64, 0, 1, false),
    // two-pass 2^19 .. 2^22 (plan.cpp build_two_pass_blocked): strips + twiddle
    // with a contiguous store, blocked rows in / transposed out
    KENTRY(8192, 16, 32, 0, 2, 1, true), KENTRYW(16384, 32, 32, 0, 1, 1, true, 2),
    KENTRYW(16384, 64, 32, 0, 1, 1, true, 2), KENTRYW(16384, 32, 32, 0, 1, 6, false, 2),
    KENTRYW(16384, 64, 32, 0, 1, 6, false, 2), KONE(16384, 32, 32, 0, 6, false), KONE(16384, 64, 32, 0, 6, false),
    // 2D split columns (plan.cpp build_2d_split_columns): pass 2a of 32 rows
    KENTRY(4096, 32, 0, 0, 4, 1, true),
    // fused distributed plans of 2^14 .. 2^18 (plan.cpp build_plan_dist): wide
    // twiddled strips and blocked rows of 128 .. 512
    KENTRY(2048, 8, 16, 0, 4, 1, true), KENTRY(2048, 8, 16, 0, 4, 6, false), KENTRY(4096, 16, 16, 0, 4, 6, false),
    KENTRY(8192, 16, 32, 0, 2, 6, false),
    // two-pass: 8192-element strips of 1024 rows (first pass); blocked rows of
    // 1024 / 2048 in 8192-element chunks (experiment TCFFT_RCHUNK_<n>)
    KENTRY(8192, 32, 32, 0, 2, 1, true), KENTRY(8192, 64, 32, 0, 2, 6, false), KENTRY(8192, 32, 32, 0, 2, 6, false),
    // column strips of 256 columns for N <= 8 (2D nx <= 8 with ny > 256)
    KSTRIP(512, 2, 0, 0, 4),      KSTRIP(1024, 4, 0, 0, 4),     KSTRIP(2048, 8, 0, 0, 4),
    // rows of 4 .. 16 whose element count is not a multiple of 32 (unswizzled staging)
    KENTRY(2048, 4, 0, 0, 4, 5, false), KENTRY(4096, 8, 0, 0, 4, 5, false), KENTRY(4096, 16, 0, 0, 4, 5, false),
    // small-batch row passes (half chunks, plan.cpp build_pass)
    KROW(2048, 16, 16, 0, 4),     KROW(2048, 16, 8, 0, 4),      KROW(2048, 8, 8, 0, 4),
};

const KernelEntry* find_kernel(const PassPlan& p) {
  int r[3] = {0, 0, 0};
  for (int s = 0; s < p.S; ++s) r[s] = p.st[s].R;
  // kPassRow 0, kPassStrip 1, kPassRowT 2 == kernel modes; strip-in / rows-out
  // passes run the strip kernel (their output addressing is all runtime)
  const int mode = p.kind == tcfft::kPassRowTB                          ? 6 /* kModeRowTB */
                   : p.kind == tcfft::kPassStripT                        ? (int)tcfft::kPassStrip
                   : (p.kind == tcfft::kPassStrip && p.out.img_split)  ? 3 /* kModeStrip4 */
                   : (p.kind == tcfft::kPassRow && p.N >= 4 && p.N < 32 && p.in.W != 32) ? 5 /* kModeRowU */
                                                                        : p.kind;
  const int tw4 = p.tw4_total ? 1 : 0;
  // the planner's warpgroup count if that instantiation exists, else one
  for (int nwg : {p.nwg, 1})
    for (const auto& k : kKernels)
      if (k.E == p.E && k.R1 == r[0] && k.R2 == r[1] && k.R3 == r[2] && k.mode == mode && k.tw4 == tw4 &&
          k.nwg == nwg && k.onebuf == p.onebuf)
        return &k;
  return nullptr;
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// Ticket counters {next, retired} per launch slot: each launch of a pass takes
// the next of kTicketSlots slots (the kernel's last CTA resets its slot), so
// up to kTicketSlots executions of one plan may be in flight concurrently on
// different streams without sharing a counter.
constexpr int kTicketSlots = 64;

struct DevPass {
  const KernelEntry* k = nullptr;
  mutable unsigned launches = 0;  // launch counter (ticket slot), atomically incremented
  void* tables = nullptr;  // rows | bblob | tblob
  KParams kp{};
  int grid = 0;
};

}  // namespace

struct HostPipe;

struct tcfftPlanImpl {
  tcfft::Plan plan;
  std::vector<DevPass> dev;
  void* ws = nullptr;
  HostPipe* pipe = nullptr;  // lazily built by tcfftExecC2CHost
  unsigned pass_mask = ~0u;  // tcfftSetPassMask (profiling)
  void* scratch = nullptr;   // strided views: contiguous staging (lazy)
  size_t scratch_bytes = 0;
  struct GraphEntry {
    const void* in;
    void* out;
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> graphs;  // grouped plans: cached per (idata, odata)
  cudaStream_t cap_stream = nullptr;
  cudaStream_t stream = nullptr;
  int device = 0;
  int magic = 0x7cff7;
};

namespace {

// L2 sector promotion of the strided (column-box) tensor maps: a box row of
// C*4 bytes fetches only its own sectors (NONE) or the whole 64/128/256-byte
// line, which the CTA working on the neighbouring strip then hits in L2
// (experiment hook TCFFT_L2PROMO = 0 / 64 / 128 / 256).
CUtensorMapL2promotion box_promotion() {
  const char* e = tcfft::experiment_env("TCFFT_L2PROMO");
  const int v = e ? std::atoi(e) : 0;
  return v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
         : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
         : v == 256 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                    : CU_TENSOR_MAP_L2_PROMOTION_NONE;
}

tcfftResult make_tmap(CUtensorMap* tm, const tcfft::IoDesc& io, const void* base) {
  std::memset(tm, 0, sizeof(*tm));
  if (io.mode == tcfft::kIoPitch || io.mode == tcfft::kIoLinear || io.mode == tcfft::kIoPeer)
    return TCFFT_SUCCESS;  // raw bulk copies
  auto enc = encode_fn();
  if (!enc) return TCFFT_EXEC_FAILED;
  CUresult r;
  if (io.mode == tcfft::kIoRank1) {
    cuuint64_t dims[1] = {(cuuint64_t)io.total};
    cuuint64_t strides[1] = {0};
    cuuint32_t box[1] = {(cuuint32_t)io.box_rows};
    cuuint32_t es[1] = {1};
    r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 1, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (io.mode == tcfft::kIoFlat) {
    cuuint64_t dims[2] = {(cuuint64_t)io.W, (cuuint64_t)(io.total / io.W)};
    cuuint64_t strides[1] = {(cuuint64_t)io.W * 4};
    cuuint32_t box[2] = {(cuuint32_t)io.W, (cuuint32_t)io.box_rows};
    cuuint32_t es[2] = {1, 1};
    r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, io.W == 32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (io.mode == tcfft::kIoFlat3) {
    cuuint64_t dims[3] = {(cuuint64_t)io.W, 256, (cuuint64_t)(io.total / io.W / 256)};
    cuuint64_t strides[2] = {(cuuint64_t)io.W * 4, (cuuint64_t)io.W * 256 * 4};
    cuuint32_t box[3] = {(cuuint32_t)io.W, 256, (cuuint32_t)io.n_sub};
    cuuint32_t es[3] = {1, 1, 1};
    // (W < 32: the contiguous store of a strip-layout staging tile, plan.cpp flat_io_w)
    const CUtensorMapSwizzle sw = io.swz == 0x70   ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : io.swz == 0x30 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : io.swz == 0x10 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                   : CU_TENSOR_MAP_SWIZZLE_NONE;
    r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (io.mode == tcfft::kIoBlk) {
    // [images][blocks][rows / C][C W]: box {C W, 1 row group, every block, 1 image}
    const int g = io.C * io.W;
    cuuint64_t dims[4] = {(cuuint64_t)g, (cuuint64_t)(io.rows / io.C), (cuuint64_t)io.cols, (cuuint64_t)io.images};
    cuuint64_t strides[3] = {(cuuint64_t)g * 4, (cuuint64_t)io.W * io.rows * 4,
                             (cuuint64_t)io.W * io.rows * io.cols * 4};
    cuuint32_t box[4] = {(cuuint32_t)g, 1, (cuuint32_t)(io.cols / io.n_sub), 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (io.mode == tcfft::kIoBoxR) {
    const int k = io.rows / 256;
    cuuint64_t dims[4] = {(cuuint64_t)io.cols, 256, (cuuint64_t)k, (cuuint64_t)io.images};
    cuuint64_t strides[3] = {(cuuint64_t)io.cols * 4, (cuuint64_t)io.cols * 256 * 4,
                             (cuuint64_t)(io.img_stride ? io.img_stride : (int64_t)io.cols * io.rows) * 4};
    cuuint32_t box[4] = {(cuuint32_t)io.C, 256, (cuuint32_t)k, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    const int run = io.C * 4;
    CUtensorMapSwizzle sw = run == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                            : run == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                            : run == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                        : CU_TENSOR_MAP_SWIZZLE_NONE;
    r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, box_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const int64_t rs = io.row_stride ? io.row_stride : io.cols;
    const int64_t is = io.img_stride ? io.img_stride : (int64_t)io.cols * io.rows;
    const int rank = io.img_split ? 4 : 3;
    cuuint64_t dims[4] = {(cuuint64_t)io.cols, (cuuint64_t)io.rows,
                          (cuuint64_t)(io.img_split ? io.img_split : io.images),
                          (cuuint64_t)(io.img_split ? io.images / io.img_split : 1)};
    cuuint64_t strides[3] = {(cuuint64_t)rs * 4, (cuuint64_t)is * 4, (cuuint64_t)io.img_stride2 * 4};
    cuuint32_t box[4] = {(cuuint32_t)io.C, (cuuint32_t)io.box_rows, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    const int run = io.C * 4;
    CUtensorMapSwizzle sw = run == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                            : run == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                            : run == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                        : CU_TENSOR_MAP_SWIZZLE_NONE;
    r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, rank, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, box_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  return r == CUDA_SUCCESS ? TCFFT_SUCCESS : TCFFT_EXEC_FAILED;
}

tcfft::KIo to_kio(const tcfft::IoDesc& io, const PassPlan& p) {
  tcfft::KIo k;
  std::memset(&k, 0, sizeof(k));
  k.mode = io.mode;
  k.box_rows = io.box_rows;
  k.n_sub = io.n_sub;
  k.sub_bytes = io.sub_bytes;
  k.chunk_rows = io.chunk_rows;
  k.C = io.C;
  k.spi = io.spi;
  k.isplit = io.img_split;
  k.pitch_bytes = p.pitch * 4;
  k.gstride_bytes = (int64_t)io.sub_bytes;  // contiguous transforms; strided exec overrides
  k.count = p.count;
  k.npeer = io.npeer;
  k.peer_blk0 = io.peer_blk0;
  return k;
}

tcfftResult map_build_status(int st) {
  switch (st) {
    case 0: return TCFFT_SUCCESS;
    case 3: return TCFFT_INVALID_VALUE;
    case 4: return TCFFT_INVALID_SIZE;
    default: return TCFFT_NOT_SUPPORTED;
  }
}

void destroy_pipe_fwd(HostPipe* hp);

// Frees everything a (possibly partially built) plan owns; shared by
// tcfftDestroy and every failure path of create().
void release(tcfftPlanImpl* h) {
  for (auto& q : h->dev) {
    if (q.tables) cudaFree(q.tables);
#ifdef TCFFT_TRACE
    if (q.kp.trace) cudaFree(q.kp.trace);
#endif
  }
  h->dev.clear();
  if (h->ws) cudaFree(h->ws);
  if (h->scratch) cudaFree(h->scratch);
  for (auto& e : h->graphs) cudaGraphExecDestroy(e.exec);
  h->graphs.clear();
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  destroy_pipe_fwd(h->pipe);
  h->ws = h->scratch = nullptr;
  h->cap_stream = nullptr;
  h->pipe = nullptr;
  h->magic = 0;
  delete h;
}

using PlanBuilder = std::function<int(tcfft::Plan&, std::string*)>;

tcfftResult create_built(tcfftHandle* out, const PlanBuilder& build);

tcfftResult create(tcfftHandle* out, int dims, int nx, int ny, int batch) {
  return create_built(out, [=](tcfft::Plan& pl, std::string* e) { return tcfft::build_plan(pl, dims, nx, ny, batch, e); });
}

tcfftResult create_built(tcfftHandle* out, const PlanBuilder& build) {
  if (!out) return TCFFT_INVALID_VALUE;
  *out = nullptr;
  auto* h = new (std::nothrow) tcfftPlanImpl();
  if (!h) return TCFFT_ALLOC_FAILED;
  std::string err;
  tcfftResult st = map_build_status(build(h->plan, &err));
  if (st != TCFFT_SUCCESS) {
    delete h;
    return st;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    delete h;
    return TCFFT_NO_DEVICE;
  }
  cudaGetDevice(&h->device);
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, h->device);
  if (prop.major != 10) {
    delete h;
    return TCFFT_NO_DEVICE;
  }
  for (const PassPlan& p : h->plan.passes) {
    DevPass d;
    d.k = find_kernel(p);
    if (!d.k) {
      release(h);
      return TCFFT_NOT_SUPPORTED;
    }
    size_t rb = p.rows_tab.size() * sizeof(tcfft::RowInfo);
    size_t bb = (p.bblob.size() * 2 + 255) & ~size_t(255);
    size_t tb = (p.tblob.size() * 4 + 255) & ~size_t(255);
    size_t rb_al = (rb + 255) & ~size_t(255);
    if (cudaMalloc(&d.tables, rb_al + bb + tb + 256 + kTicketSlots * 16) != cudaSuccess) {
      cudaGetLastError();
      release(h);
      return TCFFT_ALLOC_FAILED;
    }
    char* base = static_cast<char*>(d.tables);
    cudaMemcpy(base, p.rows_tab.data(), rb, cudaMemcpyHostToDevice);
    cudaMemcpy(base + rb_al, p.bblob.data(), p.bblob.size() * 2, cudaMemcpyHostToDevice);
    if (!p.tblob.empty()) cudaMemcpy(base + rb_al + bb, p.tblob.data(), p.tblob.size() * 4, cudaMemcpyHostToDevice);
    KParams& k = d.kp;
    std::memset(&k, 0, sizeof(k));
    k.chunks = p.chunks;
    k.T = p.T;
    k.gstride = p.gstride;
    k.ostride = p.ostride;
    k.swz_in = p.swz_in;
    k.swz_out = p.swz_out;
    k.tiles_max = p.tiles_max;
    k.in = to_kio(p.in, p);
    k.out = to_kio(p.out, p);
    k.rows_tab = reinterpret_cast<const tcfft::RowInfo*>(base);
    k.bblob = reinterpret_cast<const uint16_t*>(base + rb_al);
    k.bbytes = (int)(p.bblob.size() * 2);  // multiple of 512
    k.smem_a = p.smem_a;
    k.a_stride = p.a_bufs == 2 ? p.a_bytes : 0;
    k.smem_b = p.smem_b;
    k.smem_bar = p.smem_bar;
    k.smem_tw4 = p.smem_tw4;
    k.tw4_total = p.tw4_total;
    k.tw4_shift = p.tw4_shift;
    k.tw4_col0 = p.tw4_col0;
    k.tw4_s = p.N / p.st[p.S - 1].R;
    k.tw4_nk = k.tw4_s;
    // One-CTA-per-SM passes issue stage 1 before waiting for the previous
    // chunk's store to have read the A buffer (two-pass 2^22 second pass 0.69
    // -> 0.71 of roofline; -0.3% for the 4-CTA C2 pass, round 2)
    k.late_wait = p.ctas_per_sm == 1 ? 1 : 0;
    if (const char* e = tcfft::experiment_env("TCFFT_LATE_WAIT")) k.late_wait = std::atoi(e);
    // gather-ahead shifts when each CTA's stores land; the four-step passes
    // write 16-byte runs whose L2 merging is timing sensitive: keep them lockstep
    k.gather_ahead = (p.tw4_total || p.kind == tcfft::kPassRowT || p.kind == tcfft::kPassRowTB) ? 0 : 1;
    if (const char* e = tcfft::experiment_env("TCFFT_GATHER_AHEAD")) k.gather_ahead = std::atoi(e);
    // pipelined loop: measured faster only for the N = 1024 (32, 32) row pass
    // (0.92 vs 0.88 of roofline); slower for the 512 row pass (0.88 vs 0.97),
    // every column strip (2D 2048^2: 0.48 vs 0.60) and the twiddled passes
    // (round 1)
    k.pipe = (p.kind == tcfft::kPassRow && p.S == 2 && p.st[0].R == 32 && p.st[1].R == 32) ? 1 : 0;
    k.pdl = pdl_mode();
    // Chunk scheduling (kernel next_chunk): static striding, except that the
    // last two rounds of chunks are handed out by ticket, fetched one chunk
    // ahead, so CTAs on slower SMs take fewer of them (the static tail spread
    // was ~13 us of a 97 us C2 pass).  Measured equal or better everywhere
    // (four-step 0.80 -> 0.83, C4 +1%), round 1.  Passes with fewer than three
    // rounds stay static: the ticket + retire atomics cost short kernels (C1).
    // TCFFT_DYNAMIC=0: static; 1: tickets for every chunk after the first.
    const int dyn_mode = [] {
      const char* e = tcfft::experiment_env("TCFFT_DYNAMIC");
      return e ? std::atoi(e) : 2;
    }();
    const int64_t slots0 = (int64_t)prop.multiProcessorCount * p.ctas_per_sm;
    const int64_t grid0 = std::min<int64_t>(p.chunks, slots0);
    // (the pipelined loop takes its tickets on the critical path: static there,
    // 2D 1024^2 0.80 vs 0.73)
    const bool dyn = dyn_mode == 1 || (dyn_mode == 2 && p.chunks / grid0 >= 3 && !k.pipe);
    if (dyn) {
      k.ctr = reinterpret_cast<unsigned long long*>(base + rb_al + bb + tb + 256);
      cudaMemset(k.ctr, 0, kTicketSlots * 2 * sizeof(unsigned long long));
    }
    if (const char* e = tcfft::experiment_env("TCFFT_PDL_MASK"))
      if (!((std::atoi(e) >> h->dev.size()) & 1)) k.pdl = 0;
    if (const char* e = tcfft::experiment_env("TCFFT_PIPE")) k.pipe = std::atoi(e) && p.S >= 2 && p.kind != tcfft::kPassRowT && p.kind != tcfft::kPassRowTB;
    // the opt-in maximum: one kernel instance serves plans with different
    // shared-memory requests, occupancy follows each launch's own request
    cudaFuncSetAttribute(d.k->fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)prop.sharedMemPerBlockOptin);
    int64_t slots = (int64_t)prop.multiProcessorCount * p.ctas_per_sm;
    d.grid = (int)std::min<int64_t>(p.chunks, slots);
    k.static_chunks = d.grid;
    if (k.ctr && dyn_mode == 2) {
      static const int tail = [] {  // ticketed rounds at the end (experiment hook TCFFT_DYN_TAIL)
        const char* e = tcfft::experiment_env("TCFFT_DYN_TAIL");
        return e ? std::max(1, std::atoi(e)) : 2;
      }();
      k.static_chunks = std::max<int64_t>(d.grid, (p.chunks / d.grid - tail) * d.grid);
    }
#ifdef TCFFT_TRACE
    cudaMalloc(reinterpret_cast<void**>(&d.kp.trace), (size_t)d.grid * 8 * sizeof(unsigned long long));
#endif
    h->dev.push_back(d);
  }
  if (h->plan.ws_bytes && cudaMalloc(&h->ws, h->plan.ws_bytes) != cudaSuccess) {
    cudaGetLastError();
    release(h);
    return TCFFT_ALLOC_FAILED;
  }
  if (cudaGetLastError() != cudaSuccess) {
    release(h);
    return TCFFT_EXEC_FAILED;
  }
  *out = h;
  return TCFFT_SUCCESS;
}

bool valid(tcfftHandle h) { return h && h->magic == 0x7cff7; }

// The plan's tables, tensor maps and workspace live on the device that was
// current at plan creation: executing with another current device would read
// another GPU's memory (or fail at launch), so it is refused.
bool on_plan_device(tcfftHandle h) {
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cur == h->device;
}

}  // namespace

// bstride > 0: row-pitched batch (strided views): the first pass reads and the
// last pass writes image b at b * bstride elements (box tensor maps)
static tcfftResult launch_passes(tcfftHandle plan, const void* idata, void* odata, cudaStream_t st,
                                 int64_t bstride = 0);
static tcfftResult exec_grouped(tcfftHandle plan, const void* idata, void* odata);

extern "C" {

tcfftResult tcfftPlan1D(tcfftHandle* plan, int nx, int batch) { return create(plan, 1, nx, 0, batch); }
tcfftResult tcfftPlan2D(tcfftHandle* plan, int nx, int ny, int batch) { return create(plan, 2, nx, ny, batch); }

tcfftResult tcfftSetStream(tcfftHandle plan, void* stream) {
  if (!valid(plan)) return TCFFT_INVALID_PLAN;
  plan->stream = static_cast<cudaStream_t>(stream);
  return TCFFT_SUCCESS;
}

tcfftResult tcfftGetWorkspaceSize(tcfftHandle plan, size_t* bytes) {
  if (!valid(plan)) return TCFFT_INVALID_PLAN;
  if (!bytes) return TCFFT_INVALID_VALUE;
  *bytes = plan->plan.ws_bytes;
  return TCFFT_SUCCESS;
}

tcfftResult tcfftSetPassMask(tcfftHandle plan, unsigned mask) {
  if (!valid(plan)) return TCFFT_INVALID_PLAN;
  plan->pass_mask = mask;
  return TCFFT_SUCCESS;
}

tcfftResult tcfftExecC2C(tcfftHandle plan, const void* idata, void* odata) {
  if (!valid(plan)) return TCFFT_INVALID_PLAN;
  if (!idata || !odata || !on_plan_device(plan) || plan->plan.dist) return TCFFT_INVALID_VALUE;
  if ((reinterpret_cast<uintptr_t>(idata) | reinterpret_cast<uintptr_t>(odata)) & 15) return TCFFT_INVALID_VALUE;
  if (plan->plan.groups > 1 && plan->pass_mask == ~0u) return exec_grouped(plan, idata, odata);
  return launch_passes(plan, idata, odata, plan->stream);
}

}  // extern "C"

// All pass launches of one execution, on stream `st`.
static tcfftResult launch_passes(tcfftHandle plan, const void* idata, void* odata, cudaStream_t st, int64_t bstride) {
  for (int64_t g = 0; g < plan->plan.groups; ++g) {
  const size_t goff = (size_t)g * plan->plan.group_bytes;
  const void* src = static_cast<const char*>(idata) + goff;
  for (size_t i = 0; i < plan->dev.size(); ++i) {
    const PassPlan& p = plan->plan.passes[i];
    const DevPass& d = plan->dev[i];
    void* dst = p.ws_out ? plan->ws : static_cast<void*>(static_cast<char*>(odata) + goff);
    if (p.ws_in) src = plan->ws;
    if (!((plan->pass_mask >> i) & 1u)) {
      src = dst;
      continue;
    }
    CUtensorMap tin, tout;
    tcfft::IoDesc din = p.in, dout = p.out;
    if (bstride && i == 0) din.img_stride = bstride;
    if (bstride && i + 1 == plan->dev.size()) dout.img_stride = bstride;
    if (make_tmap(&tin, din, src) != TCFFT_SUCCESS || make_tmap(&tout, dout, dst) != TCFFT_SUCCESS)
      return TCFFT_EXEC_FAILED;
    KParams kp = d.kp;
    kp.in.gptr = static_cast<const uint8_t*>(src);
    kp.out.gptr = static_cast<const uint8_t*>(dst);
    if (kp.ctr) kp.ctr += 2 * (__atomic_fetch_add(&d.launches, 1u, __ATOMIC_RELAXED) % kTicketSlots);
    d.k->launch(dim3(d.grid), p.smem_bytes, st, tin, tout, kp);
    if (cudaGetLastError() != cudaSuccess) return TCFFT_EXEC_FAILED;
    src = dst;
  }
  }
  return TCFFT_SUCCESS;
}

// Grouped (L2-resident four-step) plans issue two launches per group: replay
// them as one CUDA graph, instantiated once per (idata, odata) pair, unless the
// caller's stream is itself being captured.
static tcfftResult exec_grouped(tcfftHandle plan, const void* idata, void* odata) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(plan->stream, &cs);
  if (cs != cudaStreamCaptureStatusNone) return launch_passes(plan, idata, odata, plan->stream);
  for (auto& e : plan->graphs)
    if (e.in == idata && e.out == odata) {
      return cudaGraphLaunch(e.exec, plan->stream) == cudaSuccess ? TCFFT_SUCCESS : TCFFT_EXEC_FAILED;
    }
  if (!plan->cap_stream && cudaStreamCreateWithFlags(&plan->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
    return TCFFT_EXEC_FAILED;
  cudaGraph_t g = nullptr;
  if (cudaStreamBeginCapture(plan->cap_stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return TCFFT_EXEC_FAILED;
  tcfftResult r = launch_passes(plan, idata, odata, plan->cap_stream);
  if (cudaStreamEndCapture(plan->cap_stream, &g) != cudaSuccess || r != TCFFT_SUCCESS) {
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    return TCFFT_EXEC_FAILED;
  }
  cudaGraphExec_t ex = nullptr;
  if (cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) {
    cudaGraphDestroy(g);
    cudaGetLastError();
    return TCFFT_EXEC_FAILED;
  }
  cudaGraphDestroy(g);
  if (plan->graphs.size() >= 4) {
    cudaGraphExecDestroy(plan->graphs.front().exec);
    plan->graphs.erase(plan->graphs.begin());
  }
  plan->graphs.push_back({idata, odata, ex});
  return cudaGraphLaunch(ex, plan->stream) == cudaSuccess ? TCFFT_SUCCESS : TCFFT_EXEC_FAILED;
}


// ---------------------------------------------------------------------------
// Host-buffer execution: the batch is cut into slices of whole transforms;
// slice i's H2D copy, transform and D2H copy run on three streams, ring of
// three device slice buffers, so both PCIe directions and the tensor-core
// kernels overlap.  Pinned host memory is needed for real overlap.
struct HostPipe {
  int64_t slice_batch = 0, slices = 0, tail = 0;
  tcfftHandle full = nullptr, last = nullptr;  // sub-plans (slice batch, tail batch)
  void* dbuf[3] = {nullptr, nullptr, nullptr};
  cudaStream_t s[3] = {nullptr, nullptr, nullptr};  // h2d, compute, d2h
  cudaEvent_t ev_in[3], ev_done[3], ev_free[3], ev_start, ev_end;
  bool ok = false;
};

static void destroy_pipe(HostPipe* hp);
namespace {
void destroy_pipe_fwd(HostPipe* hp) { destroy_pipe(hp); }
}  // namespace

static void destroy_pipe(HostPipe* hp) {
  if (!hp) return;
  if (hp->full) tcfftDestroy(hp->full);
  if (hp->last) tcfftDestroy(hp->last);
  for (int i = 0; i < 3; ++i) {
    if (hp->dbuf[i]) cudaFree(hp->dbuf[i]);
    if (hp->s[i]) cudaStreamDestroy(hp->s[i]);
    if (hp->ok) {
      cudaEventDestroy(hp->ev_in[i]);
      cudaEventDestroy(hp->ev_done[i]);
      cudaEventDestroy(hp->ev_free[i]);
    }
  }
  if (hp->ok) {
    cudaEventDestroy(hp->ev_start);
    cudaEventDestroy(hp->ev_end);
  }
  delete hp;
}

static tcfftResult build_pipe(tcfftHandle plan) {
  const tcfft::Plan& P = plan->plan;
  const int64_t n = (int64_t)P.nx * (P.dims == 2 ? P.ny : 1);
  const int64_t bytes_per = n * 4;
  auto* hp = new (std::nothrow) HostPipe();
  if (!hp) return TCFFT_ALLOC_FAILED;
  int64_t target = 16ll << 20;  // ~16 MiB slices (measured best of 8..128 MiB for C2)
  if (const char* e = tcfft::experiment_env("TCFFT_SLICE_MB")) target = std::max(1, std::atoi(e)) * (1ll << 20);
  hp->slice_batch = std::max<int64_t>(1, std::min<int64_t>(P.batch, target / bytes_per));
  hp->slices = (P.batch + hp->slice_batch - 1) / hp->slice_batch;
  hp->tail = P.batch - (hp->slices - 1) * hp->slice_batch;
  tcfftResult st = P.dims == 1 ? tcfftPlan1D(&hp->full, P.nx, (int)hp->slice_batch)
                               : tcfftPlan2D(&hp->full, P.nx, P.ny, (int)hp->slice_batch);
  if (st == TCFFT_SUCCESS && hp->tail != hp->slice_batch)
    st = P.dims == 1 ? tcfftPlan1D(&hp->last, P.nx, (int)hp->tail) : tcfftPlan2D(&hp->last, P.nx, P.ny, (int)hp->tail);
  for (int i = 0; i < 3 && st == TCFFT_SUCCESS; ++i) {
    if (cudaMalloc(&hp->dbuf[i], (size_t)(hp->slice_batch * bytes_per)) != cudaSuccess) st = TCFFT_ALLOC_FAILED;
    if (cudaStreamCreateWithFlags(&hp->s[i], cudaStreamNonBlocking) != cudaSuccess) st = TCFFT_EXEC_FAILED;
  }
  if (st == TCFFT_SUCCESS) {
    for (int i = 0; i < 3; ++i) {
      cudaEventCreateWithFlags(&hp->ev_in[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&hp->ev_done[i], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&hp->ev_free[i], cudaEventDisableTiming);
    }
    cudaEventCreateWithFlags(&hp->ev_start, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&hp->ev_end, cudaEventDisableTiming);
    hp->ok = true;
  }
  if (st != TCFFT_SUCCESS) {
    cudaGetLastError();
    destroy_pipe(hp);
    return st;
  }
  plan->pipe = hp;
  return TCFFT_SUCCESS;
}

extern "C" tcfftResult tcfftExecC2CHost(tcfftHandle plan, const void* hin, void* hout) {
  if (!valid(plan)) return TCFFT_INVALID_PLAN;
  if (plan->plan.dist) return TCFFT_INVALID_VALUE;  // distributed plans: tcfftExecDistPass
  if (!hin || !hout || !on_plan_device(plan)) return TCFFT_INVALID_VALUE;
  if (!plan->pipe) {
    tcfftResult st = build_pipe(plan);
    if (st != TCFFT_SUCCESS) return st;
  }
  HostPipe* hp = plan->pipe;
  const tcfft::Plan& P = plan->plan;
  const int64_t bytes_per = (int64_t)P.nx * (P.dims == 2 ? P.ny : 1) * 4;
  const char* src = static_cast<const char*>(hin);
  char* dst = static_cast<char*>(hout);
  if (hp->slices == 1) {  // small problem: one slice, the plan's own stream, no cross-stream events
    const size_t bytes = (size_t)(P.batch * bytes_per);
    cudaMemcpyAsync(hp->dbuf[0], src, bytes, cudaMemcpyHostToDevice, plan->stream);
    tcfftSetStream(hp->full, plan->stream);
    tcfftResult st = tcfftExecC2C(hp->full, hp->dbuf[0], hp->dbuf[0]);
    if (st != TCFFT_SUCCESS) return st;
    cudaMemcpyAsync(dst, hp->dbuf[0], bytes, cudaMemcpyDeviceToHost, plan->stream);
    return cudaGetLastError() == cudaSuccess ? TCFFT_SUCCESS : TCFFT_EXEC_FAILED;
  }
  // order after earlier work on the plan's stream
  cudaEventRecord(hp->ev_start, plan->stream);
  cudaStreamWaitEvent(hp->s[0], hp->ev_start, 0);
  for (int64_t i = 0; i < hp->slices; ++i) {
    const int b = (int)(i % 3);
    const int64_t nb = (i + 1 == hp->slices) ? hp->tail : hp->slice_batch;
    const size_t bytes = (size_t)(nb * bytes_per);
    const size_t off = (size_t)(i * hp->slice_batch * bytes_per);
    if (i >= 3) cudaStreamWaitEvent(hp->s[0], hp->ev_free[b], 0);  // slice i-3 drained
    cudaMemcpyAsync(hp->dbuf[b], src + off, bytes, cudaMemcpyHostToDevice, hp->s[0]);
    cudaEventRecord(hp->ev_in[b], hp->s[0]);
    cudaStreamWaitEvent(hp->s[1], hp->ev_in[b], 0);
    tcfftHandle sub = (nb == hp->slice_batch) ? hp->full : hp->last;
    tcfftSetStream(sub, hp->s[1]);
    tcfftResult st = tcfftExecC2C(sub, hp->dbuf[b], hp->dbuf[b]);
    if (st != TCFFT_SUCCESS) return st;
    cudaEventRecord(hp->ev_done[b], hp->s[1]);
    cudaStreamWaitEvent(hp->s[2], hp->ev_done[b], 0);
    cudaMemcpyAsync(dst + off, hp->dbuf[b], bytes, cudaMemcpyDeviceToHost, hp->s[2]);
    cudaEventRecord(hp->ev_free[b], hp->s[2]);
  }
  cudaEventRecord(hp->ev_end, hp->s[2]);
  cudaStreamWaitEvent(plan->stream, hp->ev_end, 0);
  return cudaGetLastError() == cudaSuccess ? TCFFT_SUCCESS : TCFFT_EXEC_FAILED;
}

// ---------------------------------------------------------------------------
// Strided 1D views (reference BatchedTensor, executor.py:25-51): element j of
// transform b at idata[b*batch_stride + j*stride] (complex elements).
//   stride 1, batch_stride == N          : contiguous fast path
//   stride 1, padded batch_stride (x4)   : per-transform bulk copies straight
//                                          from the padded rows (64 <= N <= 1024)
//   stride 1, batch_stride (x4), swizzled
//   row plans (N = 32, 2048 .. 8192, and
//   64 .. 256 in 4096-element chunks)     : a 3D tensor map {32, N/32, batch}
//                                          whose batch stride is the view's:
//                                          one TMA box per chunk, the same
//                                          128B-swizzled staging image as the
//                                          contiguous map (no extra HBM pass)
//   anything else                        : gather into a contiguous scratch,
//                                          transform, scatter back
__global__ void strided_copy_kernel(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, int64_t batch,
                                    int64_t n, int64_t stride, int64_t bstride, int to_contig) {
  const int64_t total = batch * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = i / n, j = i - b * n;
    const int64_t s = b * bstride + j * stride;
    if (to_contig)
      dst[i] = src[s];
    else
      dst[s] = src[i];
  }
}

extern "C" tcfftResult tcfftExecC2CStrided(tcfftHandle plan, const void* idata, void* odata, long long stride,
                                           long long batch_stride) {
  if (!valid(plan)) return TCFFT_INVALID_PLAN;
  if (plan->plan.dist) return TCFFT_INVALID_VALUE;  // distributed plans: tcfftExecDistPass
  if (!idata || !odata || !on_plan_device(plan)) return TCFFT_INVALID_VALUE;
  const tcfft::Plan& P = plan->plan;
  const int64_t n = (int64_t)P.nx * (P.dims == 2 ? P.ny : 1);
  if (stride < 1 || (P.batch > 1 && batch_stride < stride * n) || batch_stride < 1) return TCFFT_INVALID_VALUE;
  if (P.dims == 2 && stride != 1) return TCFFT_INVALID_VALUE;  // executor.py:180-181
  if (stride == 1 && batch_stride == n) return tcfftExecC2C(plan, idata, odata);
  if ((reinterpret_cast<uintptr_t>(idata) | reinterpret_cast<uintptr_t>(odata)) & 15) return TCFFT_INVALID_VALUE;
  if (P.dims == 1 && stride == 1 && (batch_stride % 4) == 0 && plan->dev.size() == 1 &&
      P.passes[0].in.mode == tcfft::kIoPitch) {
    const PassPlan& p = P.passes[0];
    const DevPass& d = plan->dev[0];
    CUtensorMap t0, t1;
    std::memset(&t0, 0, sizeof(t0));
    std::memset(&t1, 0, sizeof(t1));
    KParams kp = d.kp;
    kp.in.gptr = static_cast<const uint8_t*>(idata);
    kp.out.gptr = static_cast<const uint8_t*>(odata);
    kp.in.gstride_bytes = kp.out.gstride_bytes = batch_stride * 4;
    if (kp.ctr) kp.ctr += 2 * (__atomic_fetch_add(&d.launches, 1u, __ATOMIC_RELAXED) % kTicketSlots);
    d.k->launch(dim3(d.grid), p.smem_bytes, plan->stream, t0, t1, kp);
    return cudaGetLastError() == cudaSuccess ? TCFFT_SUCCESS : TCFFT_EXEC_FAILED;
  }
  if (P.dims == 1 && stride == 1 && (batch_stride % 4) == 0 && plan->dev.size() == 1 &&
      P.passes[0].kind == tcfft::kPassRow && P.passes[0].in.W == 32 &&
      (P.passes[0].in.mode == tcfft::kIoFlat || P.passes[0].in.mode == tcfft::kIoFlat3) && P.nx % 32 == 0 &&
      P.nx / 32 <= 256 && P.passes[0].T <= 256) {
    const PassPlan& p = P.passes[0];
    const DevPass& d = plan->dev[0];
    auto enc = encode_fn();
    if (!enc) return TCFFT_EXEC_FAILED;
    CUtensorMap tm[2];
    const void* ptr[2] = {idata, odata};
    for (int i = 0; i < 2; ++i) {
      std::memset(&tm[i], 0, sizeof(tm[i]));
      cuuint64_t dims[3] = {32, (cuuint64_t)(P.nx / 32), (cuuint64_t)P.batch};
      cuuint64_t strides[2] = {128, (cuuint64_t)batch_stride * 4};
      cuuint32_t box[3] = {32, (cuuint32_t)(P.nx / 32), (cuuint32_t)p.T};
      cuuint32_t es[3] = {1, 1, 1};
      if (enc(&tm[i], CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<void*>(ptr[i]), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return TCFFT_EXEC_FAILED;
    }
    // kernel kIoFlat3: box {32, N/32, T} at {0, 0, chunk * T} (T transforms of N * 4 bytes)
    KParams kp = d.kp;
    for (tcfft::KIo* io : {&kp.in, &kp.out}) {
      io->mode = tcfft::kIoFlat3;
      io->n_sub = p.T;
      io->sub_bytes = P.nx * 4;
    }
    if (kp.ctr) kp.ctr += 2 * (__atomic_fetch_add(&d.launches, 1u, __ATOMIC_RELAXED) % kTicketSlots);
    d.k->launch(dim3(d.grid), p.smem_bytes, plan->stream, tm[0], tm[1], kp);
    return cudaGetLastError() == cudaSuccess ? TCFFT_SUCCESS : TCFFT_EXEC_FAILED;
  }
  // two-pass plans (1D 2^15 .. 2^22) whose first pass reads and last pass
  // writes the user buffer through box tensor maps with one image per
  // transform: the image stride becomes the view's batch stride
  if (P.dims == 1 && stride == 1 && (batch_stride % 4) == 0 && P.groups == 1 && P.passes.size() == 2 &&
      P.passes[0].ws_out && P.passes[1].ws_in && plan->pass_mask == ~0u) {
    auto boxed = [&](const tcfft::IoDesc& io) {
      return (io.mode == tcfft::kIoBox || io.mode == tcfft::kIoBoxR) && io.images == P.batch && !io.img_split &&
             !io.img_stride && (int64_t)io.rows * io.cols == n;
    };
    if (boxed(P.passes[0].in) && boxed(P.passes[1].out))
      return launch_passes(plan, idata, odata, plan->stream, batch_stride);
  }
  // general view: gather -> contiguous transform -> scatter
  const size_t bytes = (size_t)(P.batch * n * 4);
  if (plan->scratch_bytes < bytes) {
    if (plan->scratch) cudaFree(plan->scratch);
    plan->scratch = nullptr;
    plan->scratch_bytes = 0;
    if (cudaMalloc(&plan->scratch, bytes) != cudaSuccess) {
      cudaGetLastError();
      return TCFFT_ALLOC_FAILED;
    }
    plan->scratch_bytes = bytes;
  }
  const int threads = 256, blocks = (int)std::min<int64_t>((P.batch * n + threads - 1) / threads, 148 * 16);
  strided_copy_kernel<<<blocks, threads, 0, plan->stream>>>(static_cast<const uint32_t*>(idata),
                                                              static_cast<uint32_t*>(plan->scratch), P.batch, n,
                                                              stride, batch_stride, 1);
  tcfftResult st = tcfftExecC2C(plan, plan->scratch, plan->scratch);
  if (st != TCFFT_SUCCESS) return st;
  strided_copy_kernel<<<blocks, threads, 0, plan->stream>>>(static_cast<const uint32_t*>(plan->scratch),
                                                              static_cast<uint32_t*>(odata), P.batch, n, stride,
                                                              batch_stride, 0);
  return cudaGetLastError() == cudaSuccess ? TCFFT_SUCCESS : TCFFT_EXEC_FAILED;
}

#ifdef TCFFT_TRACE
// trace builds only: copy pass `i`'s per-CTA stamps (start, after PDL wait,
// end, smid) of the most recent launch into `host` (grid * 4 u64)
extern "C" int tcfftDebugTrace(tcfftHandle plan, int i, void* host, size_t n) {
  if (!plan || i < 0 || i >= (int)plan->dev.size()) return -1;
  const DevPass& d = plan->dev[i];
  size_t bytes = std::min(n, (size_t)d.grid * 8 * sizeof(unsigned long long));
  cudaDeviceSynchronize();
  cudaMemcpy(host, d.kp.trace, bytes, cudaMemcpyDeviceToHost);
  return d.grid;
}
#endif

extern "C" {

tcfftResult tcfftDestroy(tcfftHandle plan) {
  if (!valid(plan)) return TCFFT_INVALID_PLAN;
  release(plan);
  return TCFFT_SUCCESS;
}

const char* tcfftGetErrorString(tcfftResult r) {
  switch (r) {
    case TCFFT_SUCCESS: return "TCFFT_SUCCESS";
    case TCFFT_INVALID_PLAN: return "TCFFT_INVALID_PLAN";
    case TCFFT_ALLOC_FAILED: return "TCFFT_ALLOC_FAILED";
    case TCFFT_INVALID_VALUE: return "TCFFT_INVALID_VALUE";
    case TCFFT_INVALID_SIZE: return "TCFFT_INVALID_SIZE";
    case TCFFT_EXEC_FAILED: return "TCFFT_EXEC_FAILED";
    case TCFFT_NOT_SUPPORTED: return "TCFFT_NOT_SUPPORTED";
    case TCFFT_NO_DEVICE: return "TCFFT_NO_DEVICE";
  }
  return "unknown tcfftResult";
}

int tcfftGetVersion(void) { return 100; }

static tcfftResult describe_json(const PlanBuilder& build, int dims, int nx, int ny, int batch, char* json,
                                 size_t cap) {
  tcfft::Plan plan;
  std::string err;
  tcfftResult st = map_build_status(build(plan, &err));
  std::string s;
  if (st != TCFFT_SUCCESS) {
    s = "{\"error\": \"" + err + "\"}";
  } else {
    s = "{\"dims\": " + std::to_string(dims) + ", \"nx\": " + std::to_string(nx) + ", \"ny\": " +
        std::to_string(ny) + ", \"batch\": " + std::to_string(batch) + ", \"ws_bytes\": " +
        std::to_string(plan.ws_bytes) + ", \"groups\": " + std::to_string(plan.groups) + ", \"passes\": [";
    for (size_t i = 0; i < plan.passes.size(); ++i) {
      const PassPlan& p = plan.passes[i];
      if (i) s += ", ";
      s += "{\"kind\": \"" + std::string(p.kind == tcfft::kPassRow ? "row" : (p.kind == tcfft::kPassStrip ? "strip" : (p.kind == tcfft::kPassStripT ? "stripT" : (p.kind == tcfft::kPassRowTB ? "rowTB" : "rowT")))) + "\", \"N\": " +
           std::to_string(p.N) + ", \"E\": " + std::to_string(p.E) + ", \"T\": " + std::to_string(p.T) +
           ", \"C\": " + std::to_string(p.C) + ", \"IMG\": " + std::to_string(p.IMG) +
           ", \"chunks\": " + std::to_string(p.chunks) + ", \"flat\": " + std::to_string(p.flat) +
           ", \"W\": " + std::to_string(p.in.W) + ", \"pitch\": " + std::to_string(p.pitch) +
           ", \"in_mode\": " + std::to_string(p.in.mode) + ", \"out_mode\": " + std::to_string(p.out.mode) +
           ", \"swz_in\": " + std::to_string(p.swz_in) + ", \"swz_out\": " + std::to_string(p.swz_out) +
           ", \"tw4_total\": " + std::to_string(p.tw4_total) + ", \"tw4_shift\": " + std::to_string(p.tw4_shift) + ", \"tw4_col0\": " + std::to_string(p.tw4_col0) + ", \"ws_in\": " + std::to_string(p.ws_in) +
           ", \"ws_out\": " + std::to_string(p.ws_out) + ", \"out_cols\": " + std::to_string(p.cols) + ", \"gstride\": " + std::to_string(p.gstride) +
           ", \"ostride\": " + std::to_string(p.ostride) + ", \"swz\": " + std::to_string(p.swz_in) +
           ", \"smem_bytes\": " + std::to_string(p.smem_bytes) + ", \"smem_a\": " + std::to_string(p.smem_a) +
           ", \"a_bytes\": " + std::to_string(p.a_bytes) + ", \"tmem_cols\": " + std::to_string(p.tmem_cols) +
           ", \"tmem_a_col\": " + std::to_string(p.tmem_a_cols) +
           ", \"ctas_per_sm\": " + std::to_string(p.ctas_per_sm) + ", \"nwg\": " + std::to_string(p.nwg) + ", \"planar0\": " + std::to_string(p.planar0) + ", \"a_bufs\": " + std::to_string(p.a_bufs) + ", \"onebuf\": " + std::to_string(p.onebuf) + ", \"kernel\": " + std::to_string(find_kernel(p) ? 1 : 0) + ", \"tiles_max\": " +
           std::to_string(p.tiles_max) + ", \"stages\": [";
      for (int sidx = 0; sidx < p.S; ++sidx) {
        const auto& t = p.st[sidx];
        if (sidx) s += ", ";
        s += "{\"R\": " + std::to_string(t.R) + ", \"n2\": " + std::to_string(t.n2) + ", \"KP\": " +
             std::to_string(t.KP) + ", \"NP\": " + std::to_string(t.NP) + ", \"tiles\": " +
             std::to_string(t.tiles) + ", \"sbo\": " + std::to_string(t.sbo) + ", \"tile_bytes\": " +
             std::to_string(t.tile_bytes) + ", \"b_off\": " + std::to_string(t.b_off) + ", \"t_off\": " +
             std::to_string(t.t_off) + ", \"hstep\": " + std::to_string(t.hstep) + ", \"im_off\": " +
             std::to_string(t.im_off) + "}";
      }
      s += "]}";
    }
    s += "]}";
  }
  if (json && cap) {
    std::strncpy(json, s.c_str(), cap - 1);
    json[cap - 1] = 0;
  }
  if (!json && cap == 0) return st;
  return s.size() < cap ? st : TCFFT_INVALID_VALUE;
}

static tcfftResult plan_tables(const PlanBuilder& build, int pass, void* rows, size_t* rows_bytes, void* bmats,
                               size_t* b_bytes, void* twid, size_t* t_bytes) {
  tcfft::Plan plan;
  std::string err;
  tcfftResult st = map_build_status(build(plan, &err));
  if (st != TCFFT_SUCCESS) return st;
  if (pass < 0 || pass >= (int)plan.passes.size()) return TCFFT_INVALID_VALUE;
  const PassPlan& p = plan.passes[pass];
  size_t rb = p.rows_tab.size() * sizeof(tcfft::RowInfo), bb = p.bblob.size() * 2, tb = p.tblob.size() * 4;
  if (rows_bytes) {
    if (rows && *rows_bytes >= rb) std::memcpy(rows, p.rows_tab.data(), rb);
    *rows_bytes = rb;
  }
  if (b_bytes) {
    if (bmats && *b_bytes >= bb) std::memcpy(bmats, p.bblob.data(), bb);
    *b_bytes = bb;
  }
  if (t_bytes) {
    if (twid && *t_bytes >= tb) std::memcpy(twid, p.tblob.data(), tb);
    *t_bytes = tb;
  }
  return TCFFT_SUCCESS;
}

tcfftResult tcfftDescribePlan(int dims, int nx, int ny, int batch, char* json, size_t cap) {
  return describe_json([=](tcfft::Plan& pl, std::string* e) { return tcfft::build_plan(pl, dims, nx, ny, batch, e); },
                       dims, nx, ny, batch, json, cap);
}

tcfftResult tcfftPlanTables(int dims, int nx, int ny, int batch, int pass, void* rows, size_t* rows_bytes,
                            void* bmats, size_t* b_bytes, void* twid, size_t* t_bytes) {
  return plan_tables([=](tcfft::Plan& pl, std::string* e) { return tcfft::build_plan(pl, dims, nx, ny, batch, e); },
                     pass, rows, rows_bytes, bmats, b_bytes, twid, t_bytes);
}

// ---- distributed single transforms (plan.cpp build_plan_dist)
tcfftResult tcfftPlan1DDist(tcfftHandle* plan, int nx, int rank, int world) {
  return create_built(plan, [=](tcfft::Plan& pl, std::string* e) { return tcfft::build_plan_dist(pl, nx, rank, world, e); });
}

tcfftResult tcfftPlan1DDistFused(tcfftHandle* plan, int nx, int rank, int world) {
  if (world > 8) return TCFFT_NOT_SUPPORTED;
  return create_built(plan,
                      [=](tcfft::Plan& pl, std::string* e) { return tcfft::build_plan_dist(pl, nx, rank, world, e, true); });
}

tcfftResult tcfftDistSetPeers(tcfftHandle plan, const void* const* recv, int world) {
  if (!valid(plan)) return TCFFT_INVALID_PLAN;
  if (plan->plan.dist != 2 || plan->plan.passes[0].out.mode != tcfft::kIoPeer || !recv ||
      world != plan->plan.passes[0].out.npeer)
    return TCFFT_INVALID_VALUE;
  for (int h = 0; h < world; ++h) {
    if (!recv[h] || (reinterpret_cast<uintptr_t>(recv[h]) & 15)) return TCFFT_INVALID_VALUE;
    plan->dev[0].kp.out.peers[h] = static_cast<const uint8_t*>(recv[h]);
  }
  return TCFFT_SUCCESS;
}

tcfftResult tcfftIpcGetHandle(const void* dptr, void* handle, size_t cap) {
  if (!dptr || !handle || cap < sizeof(cudaIpcMemHandle_t)) return TCFFT_INVALID_VALUE;
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)) != cudaSuccess) {
    cudaGetLastError();
    return TCFFT_EXEC_FAILED;
  }
  std::memcpy(handle, &h, sizeof(h));
  return TCFFT_SUCCESS;
}

tcfftResult tcfftIpcOpenHandle(const void* handle, void** dptr) {
  if (!handle || !dptr) return TCFFT_INVALID_VALUE;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  if (cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
    cudaGetLastError();
    return TCFFT_EXEC_FAILED;
  }
  return TCFFT_SUCCESS;
}

tcfftResult tcfftIpcCloseHandle(void* dptr) {
  if (!dptr) return TCFFT_INVALID_VALUE;
  return cudaIpcCloseMemHandle(dptr) == cudaSuccess ? TCFFT_SUCCESS : TCFFT_EXEC_FAILED;
}

tcfftResult tcfftDescribeDistPlanFused(int nx, int rank, int world, char* json, size_t cap) {
  return describe_json(
      [=](tcfft::Plan& pl, std::string* e) { return tcfft::build_plan_dist(pl, nx, rank, world, e, true); }, 1, nx, 0,
      1, json, cap);
}

tcfftResult tcfftDistPlanTablesFused(int nx, int rank, int world, int pass, void* rows, size_t* rows_bytes,
                                     void* bmats, size_t* b_bytes, void* twid, size_t* t_bytes) {
  return plan_tables(
      [=](tcfft::Plan& pl, std::string* e) { return tcfft::build_plan_dist(pl, nx, rank, world, e, true); }, pass, rows,
      rows_bytes, bmats, b_bytes, twid, t_bytes);
}

tcfftResult tcfftExecDistPass(tcfftHandle plan, int pass, const void* idata, void* odata) {
  if (!valid(plan)) return TCFFT_INVALID_PLAN;
  if (!plan->plan.dist || pass < 0 || pass >= (int)plan->dev.size()) return TCFFT_INVALID_VALUE;
  if (!idata || !odata || !on_plan_device(plan)) return TCFFT_INVALID_VALUE;
  if ((reinterpret_cast<uintptr_t>(idata) | reinterpret_cast<uintptr_t>(odata)) & 15) return TCFFT_INVALID_VALUE;
  const PassPlan& p = plan->plan.passes[pass];
  const DevPass& d = plan->dev[pass];
  if (p.out.mode == tcfft::kIoPeer && !d.kp.out.peers[0]) return TCFFT_INVALID_VALUE;  // tcfftDistSetPeers first
  CUtensorMap tin, tout;
  if (make_tmap(&tin, p.in, idata) != TCFFT_SUCCESS || make_tmap(&tout, p.out, odata) != TCFFT_SUCCESS)
    return TCFFT_EXEC_FAILED;
  KParams kp = d.kp;
  kp.in.gptr = static_cast<const uint8_t*>(idata);
  kp.out.gptr = static_cast<const uint8_t*>(odata);
  if (kp.ctr) kp.ctr += 2 * (__atomic_fetch_add(&d.launches, 1u, __ATOMIC_RELAXED) % kTicketSlots);
  d.k->launch(dim3(d.grid), p.smem_bytes, plan->stream, tin, tout, kp);
  return cudaGetLastError() == cudaSuccess ? TCFFT_SUCCESS : TCFFT_EXEC_FAILED;
}

tcfftResult tcfftDistUnpack(tcfftHandle plan, int world, const void* recv, void* rows) {
  if (!valid(plan)) return TCFFT_INVALID_PLAN;
  if (plan->plan.dist != 1 || world < 1 || !recv || !rows || !on_plan_device(plan)) return TCFFT_INVALID_VALUE;
  const PassPlan& p1 = plan->plan.passes[1];
  // received [G][N1/G][N2/G] (block h from rank h = columns h N2/G ..) -> rows [N1/G][N2]
  const int64_t N2 = p1.N, nrows = p1.count;
  if (N2 % world) return TCFFT_INVALID_VALUE;
  const int64_t bw = N2 / world;
  for (int h = 0; h < world; ++h) {
    const char* src = static_cast<const char*>(recv) + (size_t)h * nrows * bw * 4;
    char* dst = static_cast<char*>(rows) + (size_t)h * bw * 4;
    if (cudaMemcpy2DAsync(dst, (size_t)N2 * 4, src, (size_t)bw * 4, (size_t)bw * 4, (size_t)nrows,
                          cudaMemcpyDeviceToDevice, plan->stream) != cudaSuccess)
      return TCFFT_EXEC_FAILED;
  }
  return TCFFT_SUCCESS;
}

tcfftResult tcfftDescribeDistPlan(int nx, int rank, int world, char* json, size_t cap) {
  return describe_json([=](tcfft::Plan& pl, std::string* e) { return tcfft::build_plan_dist(pl, nx, rank, world, e); },
                       1, nx, 0, 1, json, cap);
}

tcfftResult tcfftDistPlanTables(int nx, int rank, int world, int pass, void* rows, size_t* rows_bytes, void* bmats,
                                size_t* b_bytes, void* twid, size_t* t_bytes) {
  return plan_tables([=](tcfft::Plan& pl, std::string* e) { return tcfft::build_plan_dist(pl, nx, rank, world, e); },
                     pass, rows, rows_bytes, bmats, b_bytes, twid, t_bytes);
}

}  // extern "C"
