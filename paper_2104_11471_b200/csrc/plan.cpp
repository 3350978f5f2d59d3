// plan.cpp - host-side planner (see plan.hpp).  Pure C++, no CUDA calls, so the
// same tables can be built and checked on a CPU-only machine.
//
// Algorithm (reference pkg/src/tcfft/kernels.py:323-356, plan.py:141-158): the
// transform is N = R_1 * R_2 * ... * R_S.  Stage s combines R_s sub-spectra of
// length n2_s = R_1..R_{s-1}.  With the reference's digit-reversed positions
// p = k + n2*m + n2*R*blk, stage s butterfly (k, blk) reads input m = d_s and
// writes output j; its input m carries twiddle W_{R n2}^{m k}.  Stage 1 reads
// natural-order input x[m*N/R_1 + b] directly (digit reversal folded into the
// gather addresses); the last stage writes X[k + (N/R_S) j] in natural order.
#include "plan.hpp"

#include <cmath>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>

namespace tcfft {

namespace {

uint16_t f64_to_f16_rne(double x) {
  // IEEE binary16, round to nearest even, with subnormals and overflow to inf.
  uint16_t sign = std::signbit(x) ? 0x8000 : 0;
  double a = std::fabs(x);
  if (std::isnan(x)) return 0x7e00;
  if (a >= 65520.0) return sign | 0x7c00;
  if (a < std::ldexp(1.0, -25)) {
    // below half the smallest subnormal (ties at exactly 2^-25 round to even 0)
    return sign;
  }
  int e;
  double m = std::frexp(a, &e);  // a = m * 2^e, m in [0.5, 1)
  int exp16 = e - 1 + 15;        // biased exponent for 1.xxx * 2^(e-1)
  if (exp16 <= 0) {
    // subnormal: value = q * 2^-24
    double q = a * std::ldexp(1.0, 24);
    double r = std::nearbyint(q);  // default rounding mode: nearest-even
    return sign | (uint16_t)r;
  }
  double frac = (m * 2.0 - 1.0) * 1024.0;  // 10-bit mantissa, fractional
  double r = std::nearbyint(frac);
  uint32_t mant = (uint32_t)r;
  if (mant == 1024) {
    mant = 0;
    exp16 += 1;
    if (exp16 >= 31) return sign | 0x7c00;
  }
  return sign | (uint16_t)(exp16 << 10) | (uint16_t)mant;
}

double f16_to_f64(uint16_t h) {
  int s = h >> 15, e = (h >> 10) & 31, m = h & 1023;
  double v;
  if (e == 0)
    v = std::ldexp((double)m, -24);
  else if (e == 31)
    v = m ? NAN : INFINITY;
  else
    v = std::ldexp(1.0 + m / 1024.0, e - 15);
  return s ? -v : v;
}

// W_n^e = exp(-2 pi i e / n) with the exponent reduced exactly first
// (reference twiddle.py:21-42).
void root(int64_t e, int64_t n, double* re, double* im) {
  int64_t r = ((e % n) + n) % n;
  double ang = -2.0 * M_PI * (double)r / (double)n;
  *re = std::cos(ang);
  *im = std::sin(ang);
}

struct Bf {
  int32_t tr, k, blk;
};

}  // namespace

const char* experiment_env(const char* name) {
  const char* e = std::getenv("TCFFT_EXPERIMENTS");
  return (e && std::atoi(e) == 1) ? std::getenv(name) : nullptr;
}

int writer_groups(int R, int rows_next) {
  if (R == 32 && rows_next >= 8 * R) return 8;  // (same reason as radix 64 below: 16-column strips)
  if (R <= 32) return kLanes / R;
  // a super-block of G groups x R rows must fit the next stage.  Eight groups
  // when they fit: the 8 lanes of a quarter-warp (8 columns of one butterfly
  // in 8-column strips) then store to 8 consecutive padded row blocks, 8
  // distinct 16-byte bank groups; with 4 groups rows g and g + 32 share banks
  // (2-way conflicted writer stores, round 2 ncu: 4.2M excess wavefronts in
  // the C3 strip pass)
  if (rows_next >= 8 * R) return 8;
  return rows_next >= 4 * R ? 4 : 2;
}

// experiment hook: TCFFT_ROW4096_R64=1 plans 4096-point rows as [64, 64] in
// 8192-element chunks (two stages, shared planar DFT matrix)
static bool row4096_r64() {
  const char* e = experiment_env("TCFFT_ROW4096_R64");
  return e && std::atoi(e) != 0;
}

static bool strip_quarter_order() {
  const char* e = experiment_env("TCFFT_STRIP_QUARTER");
  return !e || std::atoi(e) != 0;
}

// Strip-in / rows-out output staging pad (words).  0 = dense [column][k]
// tile written by ONE TMA store per chunk (final stores 2-way conflicted for
// N <= 128, 4-way for N = 256); a pad of 8 makes them conflict-free but needs
// one bulk copy per row: measured 23.3 vs 20.6 TFLOP/s for C3 (N = 128,
// round 1), so dense unless the conflicts get worse than 2-way.
static int pitch_pad_words_out(int n) {
  const char* e = experiment_env("TCFFT_STRIPT_PAD");
  if (e) return std::atoi(e);
  return n <= 128 ? 0 : 8;
}

int pitch_pad_words(int n) {
  // chosen with tests/emulator.py's bank model (see test_plan_emulation.py)
  const char* e = experiment_env("TCFFT_PITCH_PAD");
  if (e) return std::atoi(e);
  return (n >= 64 && n <= 1024) ? 8 : 0;
}

std::vector<int> choose_radices(int n, int kind, bool twiddled) {
  // Strided passes (column strips, transposed rows) of 2048 / 4096 use two
  // stages with a radix-64 first stage: with three stages the final stage's
  // 8-row groups hold outputs k, k + 16, ... of one butterfly, which in the
  // 4-column (16 B) strip / 4-row transposed staging all fall into one bank
  // (8-way conflicted output stores, tests/emulator.py).  With two stages the
  // final k run is consecutive.  Radix-64 stage 1 reads its A operand from
  // TMEM, so the larger DFT block costs no extra shared-memory traffic.
  const char* e = experiment_env("TCFFT_STRIDED_R64");
  const bool r64 = !e || std::atoi(e) != 0;
  if (kind != kPassRow && r64) {
    if (n == 2048) return {64, 32};
    if (n == 4096) return {64, 64};
  }
  // Plain column strips of 512 / 1024 (2D, 8192-element chunks): a radix-64
  // last stage (fewer, larger MMA tiles, one 64-output epilogue per lane):
  // C4 +1% (round 1).
  // TCFFT_STRIP_R64=0 restores [16, 32] / [32, 32].
  if (kind == kPassRow && n == 4096 && row4096_r64()) return {64, 64};
  // Strided 128-point passes: [8, 16] (two final tiles of 16 outputs per lane
  // instead of four of 8: fewer per-tile twiddle setups; C3 +2%, round 1).
  // TCFFT_STRIP128=0 restores [16, 8].
  if (kind != kPassRow && n == 128) {
    const char* e3 = experiment_env("TCFFT_STRIP128");
    if (!e3 || std::atoi(e3) != 0) return {8, 16};
  }
  // experiment hook: TCFFT_RADICES_<n>=a,b[,c] overrides a row pass's radix list
  // (needs a matching kernel instantiation; the 16384 / 8192 alternatives were
  // measured no better, profiles/exp_radix_r02.txt)
  if (kind == kPassRow) {
    char key[40];
    std::snprintf(key, sizeof(key), "TCFFT_RADICES_%d", n);
    if (const char* ev = experiment_env(key)) {
      std::vector<int> r;
      for (const char* q = ev; *q;) {
        r.push_back(std::atoi(q));
        while (*q && *q != ',') ++q;
        if (*q == ',') ++q;
      }
      return r;
    }
  }
  // (2D column strips 1024^2: 0.75 -> 0.83 of roofline)
  if (kind == kPassStrip && !twiddled && (n == 512 || n == 1024)) {
    const char* e2 = experiment_env("TCFFT_STRIP_R64");
    const int v = e2 ? std::atoi(e2) : 1;
    if (v) return n == 512 ? std::vector<int>{8, 64} : std::vector<int>{16, 64};
  }
  switch (n) {
    case 2: return {2};
    case 4: return {4};
    case 8: return {8};
    case 16: return {16};
    case 32: return {32};
    case 64: return {8, 8};
    case 128: return {16, 8};
    case 256: return {16, 16};
    case 512: return {16, 32};
    case 1024: return {32, 32};
    case 2048: return {16, 16, 8};
    case 4096: return {16, 16, 16};
    case 8192: return {16, 16, 32};
    case 16384: return {16, 32, 32};
    default: return {};
  }
}

int chunk_elems_for(int n) {
  // experiment hook: TCFFT_CHUNK_<n>=<elems> overrides the chunk size
  char key[32];
  std::snprintf(key, sizeof(key), "TCFFT_CHUNK_%d", n);
  if (const char* e = experiment_env(key)) return std::atoi(e);
  if (n <= 2) return 1024;
  if (n == 4) return 2048;
  if (n == 4096 && row4096_r64()) return 8192;
  if (n <= 4096) return 4096;
  return n;  // 8192, 16384: one transform per chunk
}

// Flat (contiguous chunk) TMA view of `total` elements.
static void flat_io(IoDesc& io, int64_t total, int E, bool allow_swizzle) {
  // W = 32: [total/32][32] view, 128B swizzle; W = 4: [total/4][4];
  // W = 1: rank-1 view [total] in 256-element boxes (any total).
  const bool can32 = (total % 32 == 0) && allow_swizzle;
  io.W = can32 ? 32 : (total % 4 == 0 ? 4 : 1);
  io.mode = io.W == 1 ? kIoRank1 : kIoFlat;
  io.swz = io.W == 32 ? 0x70 : 0;
  io.box_rows = std::min(E / io.W, 256);
  io.n_sub = (E / io.W) / io.box_rows;
  io.sub_bytes = io.box_rows * io.W * 4;
  io.chunk_rows = E / io.W;
  io.total = total;
  // chunks of more than 256 rows: one 3D box instead of n_sub 2D boxes
  const char* e = experiment_env("TCFFT_FLAT3");
  if (io.mode == kIoFlat && io.n_sub > 1 && (total / io.W) % 256 == 0 && (!e || std::atoi(e) != 0))
    io.mode = kIoFlat3;
}

// 3D column-box TMA view of an images x rows x cols array, C columns per chunk.
static void box_io(IoDesc& io, int64_t images, int rows, int cols, int C) {
  io.mode = kIoBox;
  io.images = images;
  io.rows = rows;
  io.cols = cols;
  io.C = C;
  io.spi = cols / C;
  const int run = C * 4;
  io.swz = run == 128 ? 0x70 : run == 64 ? 0x30 : run == 32 ? 0x10 : 0;
  io.box_rows = std::min(rows, 256);
  io.n_sub = rows / io.box_rows;
  io.sub_bytes = io.box_rows * C * 4;
  // strips of more than 256 rows: one 4D box ({C, 256, rows/256, 1}) per chunk
  // instead of rows/256 boxes (TCFFT_BOXR=0 keeps the sub-boxes)
  const char* e = experiment_env("TCFFT_BOXR");
  if (rows > 256 && (!e || std::atoi(e) != 0)) {
    io.mode = kIoBoxR;
    io.n_sub = 1;
    io.sub_bytes = rows * C * 4;
  }
}

// The staging tile of a chunk, byte for byte (its swizzle included), to
// elements [c E, (c + 1) E): one non-tensor bulk copy per chunk (two-pass
// plans store the first pass's column-strip tiles this way; a tensor map of
// the strip's 32-byte rows would cost one TMA request per row).
static void linear_io(IoDesc& io, int64_t total, int E, int swz) {
  io.mode = kIoLinear;
  io.W = 0;
  io.swz = swz;
  io.n_sub = 1;
  io.sub_bytes = E * 4;
  io.total = total;
}

// DFT block matrices of every stage, fp16, UMMA K-major core-matrix order.
// Full: the real 2R x 2R matrix [[Fr, Fi], [-Fi, Fr]] (K = (m, re/im), N =
// (j, re/im)); stages with the same radix and planar K share one copy
// (kernel Cfg::BOFF).
static void build_bblob(PassPlan& p) {
  const bool planar0 = p.planar0 != 0;
  p.bblob.clear();
  auto planar = [&](int s) { return s >= 1 || planar0; };
  auto put = [&](int K, int N, auto val) {  // K x N matrix, K-major canonical layout
    std::vector<uint16_t> blob(K * N, 0);
    for (int k = 0; k < K; ++k)
      for (int n = 0; n < N; ++n) {
        int q = k / 16, kk = k % 16;
        size_t off = (size_t)q * 32 * N + (n % 8) * 16 + (n / 8) * 256 + (kk / 8) * 128 + (kk % 8) * 2;
        blob[off / 2] = f64_to_f16_rne(val(k, n));
      }
    p.bblob.insert(p.bblob.end(), blob.begin(), blob.end());
  };
  auto F = [&](int R, int j, int m, bool im) {
    double fr, fi;
    root((int64_t)j * m, R, &fr, &fi);
    return f16_to_f64(f64_to_f16_rne(im ? fi : fr));  // fp16 like the reference's dft_matrix
  };
  for (int s = 0; s < p.S; ++s) {
    StageInfo& st = p.st[s];
    const int R = st.R, KP = st.KP, NP = st.NP;
    st.b_bytes = KP * NP * 2;
#ifndef TCFFT_NO_BDEDUPE
    if (s >= 1 && planar(s) && planar(s - 1) && p.st[s - 1].R == R) {  // identical planar-K matrix: share it
#else
    if (false) {
#endif
      st.b_off = p.st[s - 1].b_off;
      continue;
    }
    st.b_off = (int)(p.bblob.size() * 2);
    put(KP, NP, [&](int k, int n) {
      if (k >= 2 * R || n >= 2 * R) return 0.0;
      int m, cin;
      if (s == 0 && !planar0) {
        m = k / 2;
        cin = k % 2;
      } else {
        m = k % R;
        cin = k / R;
      }
      const int j = n % R, cout = n / R;
      const double fr = F(R, j, m, false), fi = F(R, j, m, true);
      if (cin == 0 && cout == 0) return fr;
      if (cin == 1 && cout == 0) return -fi;
      if (cin == 0 && cout == 1) return fi;
      return fr;
    });
  }
}

bool build_pass(PassPlan& p, int kind, int N, int64_t count, int64_t images, int cols, std::string* err,
                int64_t tw4_total, int tw4_shift, int blk, int want_E) {
  std::vector<int> rad = choose_radices(N, kind, tw4_total != 0);
  if (rad.empty()) {
    if (err) *err = "no single-pass radix schedule for N=" + std::to_string(N);
    return false;
  }
  p = PassPlan();
  p.kind = kind;
  p.N = N;
  p.S = (int)rad.size();
  p.tw4_total = tw4_total;
  p.tw4_shift = tw4_shift;
  const bool row_in = kind == kPassRow || kind == kPassRowT;
  const bool blk_in = kind == kPassRowTB;  // rows of a blocked array (runtime gather addressing)
  if (kind == kPassRow) {
    p.E = chunk_elems_for(N);
    // Small batches (fewer 4096-element chunks than 4 CTA slots on every SM)
    // are latency bound: halve the chunk so each CTA's load -> 2 MMA stages ->
    // store chain is shorter and twice as many CTAs share the work (C1
    // N=256 x 4096: 7.2 -> 8.1 TFLOP/s, round 1).
    const char* ce = experiment_env("TCFFT_SMALL_CHUNK");
    if ((!ce || std::atoi(ce) != 0) && p.E == 4096 && N >= 64 && N <= 256 &&
        (count * (int64_t)N + 4095) / 4096 < 148 * 4)
      p.E = 2048;
    p.T = p.E / N;
    p.count = count;
    p.chunks = (count + p.T - 1) / p.T;
  } else if (kind == kPassRowT || kind == kPassRowTB) {
    // rows of an images x (count/images) x N array, output transposed into
    // images x N x (count/images): >= 4 rows per chunk (>= 16 B output runs)
    p.E = want_E ? want_E : std::max(chunk_elems_for(N), 4 * N);
    {
      char key[32];  // experiment hook: TCFFT_RCHUNK_<n>=<elems> overrides the transposed-row chunk size
      std::snprintf(key, sizeof(key), "TCFFT_RCHUNK_%d", N);
      if (const char* e = experiment_env(key)) p.E = std::atoi(e);
    }
    p.T = p.E / N;
    p.count = count;
    p.chunks = (count + p.T - 1) / p.T;
    p.images = images;
    p.cols = (int)(count / images);  // rows per image = output columns
    if ((p.cols % p.T) != 0) {
      if (err) *err = "transposed row pass: rows per image must be a multiple of the chunk";
      return false;
    }
  } else {
    // Column strips of an images x N x cols array: C columns of IMG images per
    // chunk, E = N * C * IMG = max(chunk_elems_for(N), 4 N) (C >= 4: >= 16 B runs).
    // (>= 4 columns: TMA boxes move >= 16 bytes per row, so 2D columns of
    // 8192+ rows would need 128 KB chunks: not supported)
    p.E = want_E ? want_E : std::max(chunk_elems_for(N), 4 * N);
    // Plain column strips (2D) of 512 .. 2048 use wider chunks: C = 16 / 8 / 8
    // columns (64 / 32 / 32-byte runs) instead of 8 / 4 / 4.  Measured with
    // the lock-step loop: 2D 512^2 0.80 -> 0.88, 1024^2 0.57 -> 0.83 of the
    // HBM roofline (round 1).  Twiddled (four-step) strips keep 4096.
    if (kind == kPassStrip && !tw4_total && !want_E && (N == 512 || N == 1024)) p.E = 8192;
    if (kind == kPassStrip && !tw4_total && !want_E && N == 2048) p.E = 16384;
    {
      char key[32];  // experiment hook: TCFFT_SCHUNK_<n>=<elems> overrides the strip chunk size
      std::snprintf(key, sizeof(key), "TCFFT_SCHUNK_%d", N);
      if (const char* e = experiment_env(key)) p.E = std::atoi(e);
    }
    int ci = p.E / N;  // C * IMG
    if (ci <= cols) {
      p.C = ci;
      p.IMG = 1;
    } else {
      p.C = cols;
      p.IMG = ci / cols;
    }
    if (p.C < cols && p.C > 256) {
      // TMA boxes hold <= 256 columns: short columns (N <= 8) of wide images
      // take 256-column strips, i.e. smaller chunks
      p.C = 256;
      p.E = 256 * N;
    }
    p.T = p.C * p.IMG;
    p.images = images;
    p.rows = N;
    p.cols = cols;
    p.count = images * (int64_t)cols;
    p.chunks = (images + p.IMG - 1) / p.IMG * (int64_t)(cols / p.C);
  }
  const int E = p.E, T = p.T, S = p.S;
  const int C = p.C, NN = N;
  if (E < 128 * rad[0] || E > 16384) {
    if (err) *err = "unsupported chunk size";
    return false;
  }
  // Contiguous row inputs with 64 <= N <= 1024 stage each transform at a padded
  // pitch (per-transform bulk copies) so that the lanes of a warp, which span
  // several short transforms, fall into different shared-memory banks.
  // (kernel Cfg::PITCH mirrors this: rows of 64 .. 256 in 4096-element chunks
  // use the flat swizzled map instead)
  p.pitch_mode = row_in && N >= 64 && N <= 1024 && !(N <= 256 && p.E == 4096);
  // strip-in / rows-out passes may stage their output rows at a padded pitch
  // (pitch_pad_words_out)
  p.pitch = p.pitch_mode ? N + pitch_pad_words(N) : (kind == kPassStripT ? N + pitch_pad_words_out(N) : N);  // words
  const int PW = p.pitch;
  if (blk_in && (blk <= 0 || N % blk || (N / rad[0]) % blk)) {
    if (err) *err = "blocked rows: block width must divide N / R1";
    return false;
  }
  auto w_in = [&](int tr, int n) -> int32_t {
    // blocked rows: element n of row tr at (n / Bw) (Bw T) + tr Bw + n % Bw
    if (blk_in) return (n / blk) * (blk * T) + tr * blk + n % blk;
    return row_in ? tr * PW + n : (tr / C) * NN * C + n * C + tr % C;
  };
  auto w_out = [&](int tr, int n) -> int32_t {
    if (kind == kPassRow) return tr * PW + n;
    if (kind == kPassStripT) return tr * PW + n;
    if (kind == kPassRowT || kind == kPassRowTB) return n * T + tr;
    return (tr / C) * NN * C + n * C + tr % C;
  };
  p.gstride = (N / rad[0]) * (blk_in ? T : (row_in ? 1 : C));
  p.ostride = (N / rad[S - 1]) *
              (kind == kPassRow || kind == kPassStripT ? 1 : (kind == kPassRowT || kind == kPassRowTB ? T : C));

  // ---- TMA / bulk-copy descriptors
  if (blk_in) {
    // images x blocks x rows x Bw: one 4D box {T Bw, 1, all blocks, 1} per
    // chunk (T-row groups of every block: Bw * T * 4-byte runs)
    const int rows = (int)(count / images);
    p.in.mode = kIoBlk;
    p.in.W = blk;
    p.in.rows = rows;
    p.in.cols = N / blk;
    p.in.images = images;
    p.in.C = T;
    p.in.spi = rows / T;
    // (more than 256 blocks: boxes of 256 blocks each, consecutive in SMEM)
    p.in.n_sub = (N / blk + 255) / 256;
    p.in.sub_bytes = E * 4 / p.in.n_sub;
    p.in.box_rows = (N / blk) / p.in.n_sub;  // blocks per box
    p.in.swz = 0;
    p.in.total = count * (int64_t)N;
    if ((N / blk) % p.in.n_sub || T * blk > 256 || rows % T) {
      if (err) *err = "blocked rows: unsupported geometry";
      return false;
    }
  } else if (row_in) {
    const int64_t total = count * (int64_t)N;
    if (p.pitch_mode) {
      p.in.mode = kIoPitch;
      p.in.swz = 0;
      p.in.n_sub = T;
      p.in.sub_bytes = N * 4;
      p.in.total = total;
    } else {
      // 128B-swizzled [total/32][32] view for N >= 4 (kernel Cfg::SWZ mirrors
      // this; N = 2 keeps the plain view)
      flat_io(p.in, total, E, N >= 4);
    }
  } else if (p.C == cols) {
    flat_io(p.in, images * (int64_t)N * cols, E, true);
  } else {
    box_io(p.in, images, N, cols, C);
  }
  if (kind == kPassRowT || kind == kPassRowTB) {
    box_io(p.out, images, N, p.cols, T);
  } else if (kind == kPassStripT && PW == N) {
    flat_io(p.out, images * (int64_t)N * cols, E, true);  // unpadded: one TMA store per chunk
  } else if (kind == kPassStripT) {
    // chunk (image, strip) -> C contiguous rows of N at chunk * E, one bulk
    // copy per row from the padded staging pitch
    p.out.mode = kIoPitch;
    p.out.swz = 0;
    p.out.n_sub = T;
    p.out.sub_bytes = N * 4;
    p.out.total = images * (int64_t)N * cols;
  } else {
    p.out = p.in;
  }
  p.swz_in = p.in.swz;
  p.swz_out = p.out.swz;
  p.flat = p.in.mode != kIoBox && p.in.mode != kIoBoxR;
  p.total = p.in.total;

  int n2 = 1, tiles_max = 0;
  for (int s = 0; s < S; ++s) {
    StageInfo& st = p.st[s];
    st.R = rad[s];
    st.n2 = n2;
    n2 *= rad[s];
    st.KP = std::max(2 * st.R, 16);
    st.NP = std::max(2 * st.R, 16);
    if (E % (kLanes * st.R)) {
      if (err) *err = "chunk not a whole number of tiles";
      return false;
    }
    st.tiles = E / (kLanes * st.R);
    tiles_max = std::max(tiles_max, st.tiles);
    if (s > 0 && st.R < 8) {
      if (err) *err = "radix < 8 only supported as a single stage";
      return false;
    }
    st.sbo = 32 * st.R + 16;
    st.tile_bytes = 16 * st.sbo;
    st.t_off = -1;
    st.hstep = st.im_off = 0;
  }
  p.tiles_max = tiles_max;

  // ---- row identities per stage, writer tables -------------------------
  p.rows_tab.assign((size_t)S * tiles_max * kLanes, RowInfo{});
  auto rec = [&](int s, int row) -> RowInfo& {
    return p.rows_tab[((size_t)s * tiles_max + row / kLanes) * kLanes + row % kLanes];
  };
  // stage-1 butterflies: blk in [0, N/R1); natural base b(blk)
  const int R1 = rad[0];
  std::vector<int> P(S);
  for (int i = 0; i < S; ++i) {
    int prod = 1;
    for (int l = i + 1; l < S; ++l) prod *= rad[l];
    P[i] = prod;
  }
  auto bnat = [&](int blk) {
    int b = 0, rem = blk;
    for (int i = 1; i < S; ++i) {
      int d = rem % rad[i];
      rem /= rad[i];
      b += d * P[i];
    }
    return b;
  };
  std::vector<Bf> cur;
  cur.reserve(E / R1);
  {
    std::vector<std::tuple<int32_t, int, int>> order;
    // Rows in staging-address order (conflict-free 4-byte gathers).  Strip
    // passes with 4-column strips instead give each quarter-warp 8 consecutive
    // butterflies of one column (still 32 distinct banks for the gather, since
    // a row of the strip is 4 words): the radix-64 writer's 16-byte stores of
    // a quarter-warp then cover 128 contiguous bytes.
    const bool quarter = !row_in && C == 4 && strip_quarter_order();
    // Blocked-row inputs: the rows of a butterfly fastest (key n T + tr).  A
    // warp still covers every (row, n % Bw) bank of its block group for the
    // gather, and a quarter-warp (8 rows of one butterfly) stores the radix-64
    // writer's vectors to 8 consecutive padded row blocks (staging-address
    // order put 2 rows x 4 butterflies there: 2-way conflicts at Bw = 4)
    const char* ebo = experiment_env("TCFFT_BLK_ORDER");  // experiment: 0 = staging-address order
    const bool rows_fast = blk_in && (!ebo || std::atoi(ebo) != 0);
    for (int tr = 0; tr < T; ++tr)
      for (int blk = 0; blk < N / R1; ++blk) {
        const int n = bnat(blk);
        const int32_t key = rows_fast ? n * T + tr : quarter ? (((n / 8) * C + tr) * 8 + n % 8) : w_in(tr, n);
        order.emplace_back(key, tr, blk);
      }
    std::sort(order.begin(), order.end());
    for (auto& o : order) cur.push_back(Bf{std::get<1>(o), 0, std::get<2>(o)});
  }
  for (size_t i = 0; i < cur.size(); ++i) rec(0, (int)i).gbase = w_in(cur[i].tr, bnat(cur[i].blk));

  for (int s = 0; s + 1 < S; ++s) {
    StageInfo& st = p.st[s];
    StageInfo& nx_ = p.st[s + 1];
    // G = groups of R next-stage rows interleaved block-wise (8-row blocks:
    // block h of group g at row block (g / G) * G * R/8 + g % G + G * h).  At
    // least 4, so that a warp's 32 rows come from 4 different groups (radix-64
    // writers otherwise put 2 groups x 16 consecutive outputs in a warp: 2-way
    // conflicted strided output stores).  The A region is linear in the row
    // block (tile_bytes == 16 * sbo), so a super-block may span tiles.
    const int R = st.R, Rn = nx_.R, G = writer_groups(R, E / Rn);
    const int n2n = st.n2 * R;  // n2 of the next stage
    std::map<std::tuple<int, int, int>, int> gid;
    std::vector<Bf> nxt(E / Rn);
    st.hstep = G * nx_.sbo;
    st.im_off = Rn * 16;
    for (size_t rho = 0; rho < cur.size(); ++rho) {
      const Bf& w = cur[rho];
      int mp = w.blk % Rn, blkn = w.blk / Rn;
      auto key = std::make_tuple(w.tr, w.k, blkn);
      auto it = gid.find(key);
      int g;
      if (it == gid.end()) {
        g = (int)gid.size();
        gid.emplace(key, g);
        for (int j = 0; j < R; ++j) {
          int idx = (g / G) * G * R + ((g % G) + G * (j / 8)) * 8 + j % 8;
          nxt[idx] = Bf{w.tr, w.k + st.n2 * j, blkn};
        }
      } else {
        g = it->second;
      }
      RowInfo& r = rec(s, (int)rho);
      r.addr = ((g / G) * G * (R / 8) + (g % G)) * nx_.sbo + mp * 16;
      r.mp = mp;
      r.tw = s > 0 ? 1 : 0;
      double cr, ci, wr, wi;
      root((int64_t)mp * w.k, (int64_t)Rn * n2n, &cr, &ci);
      root((int64_t)mp, (int64_t)Rn * R, &wr, &wi);
      r.cr = (float)cr;
      r.ci = (float)ci;
      r.wr = (float)wr;
      r.wi = (float)wi;
    }
    cur.swap(nxt);
  }
  for (size_t i = 0; i < cur.size(); ++i) {
    RowInfo& r = rec(S - 1, (int)i);
    r.addr = w_out(cur[i].tr, cur[i].k);
    if (tw4_total) {
      // four-step twiddle W_Ntot^{n2 k1}, n2 = strip base + tr, k1 = k + (N/R_S) j:
      // host part W^{tr k} * (W^{tr s})^j, s = N/R_S; the strip-base part is
      // rebuilt per chunk on the device (kernel tw4 tables).
      // With tw4_shift (three-step pass B, 2D split columns) the exponent is
      // (column >> shift) * k1; chunks start at multiples of C (powers of
      // two), so (base + tr) >> shift = (base >> shift) + (tr >> shift).
      const int64_t s_ = N / rad[S - 1];
      const int64_t trx = cur[i].tr >> tw4_shift;
      double cr, ci, wr, wi;
      root(trx * cur[i].k, tw4_total, &cr, &ci);
      root(trx * s_, tw4_total, &wr, &wi);
      r.mp = cur[i].k;
      r.cr = (float)cr;
      r.ci = (float)ci;
      r.wr = (float)wr;
      r.wi = (float)wi;
    }
  }

  // ---- B matrices ---------------------------------------------------------
  // radix-64 first stages use a planar-K TMEM A operand (kernel Cfg::PLANAR0)
  const bool planar0 = rad[0] == 64;
  p.planar0 = planar0 ? 1 : 0;
  build_bblob(p);
  p.tblob.clear();  // twiddles come from the per-row (c, w) recurrence

  // ---- shared memory / TMEM budget ---------------------------------------
  const int stage_bytes = row_in ? T * PW * 4 : E * 4;                            // input staging
  const int out_bytes = (row_in || kind == kPassStripT) ? T * PW * 4 : E * 4;     // output staging (A buffer)
  {
    int acols = p.st[0].tiles * (p.st[0].KP / 2), dcols = 0;
    for (int s2 = 0; s2 < S; ++s2) dcols = std::max(dcols, p.st[s2].tiles * p.st[s2].NP);
    int need = acols + dcols, tc = 32;
    while (tc < need) tc <<= 1;
    p.tmem_cols_needed = tc;
  }
  const int tw4_bytes = tw4_total ? ((N / rad[S - 1]) * 8 + 16 + 127) & ~127 : 0;
  int a_bytes = std::max(stage_bytes, out_bytes);
  for (int s = 1; s < S; ++s) a_bytes = std::max(a_bytes, p.st[s].tiles * p.st[s].tile_bytes);
  a_bytes = (a_bytes + 1023) & ~1023;
  p.a_bytes = a_bytes;
  p.smem_in = 0;
  p.smem_a = (stage_bytes + 1023) & ~1023;
  // two A / output-staging buffers: chunk i's epilogues never wait for the TMA
  // store of chunk i-1 to finish reading its staging tile
  // (only when that still leaves room for the TMEM-limited number of CTAs/SM)
  {
    const int fixed = p.smem_a + a_bytes + (((int)p.bblob.size() * 2 + 127) & ~127) + tw4_bytes + 64 + 1024;
    const int tmem_ctas = std::max(1, 512 / std::max(32, p.tmem_cols_needed));
#ifdef TCFFT_PINGPONG
    p.a_bufs = (fixed + a_bytes + 1024) * std::min(tmem_ctas, 4) <= 233472 ? 2 : 1;
#else
    p.a_bufs = 1;
    (void)fixed;
    (void)tmem_ctas;
#endif
    if (const char* e = experiment_env("TCFFT_ABUFS")) p.a_bufs = std::max(1, std::min(2, std::atoi(e)));
  }
  p.smem_b = p.smem_a + p.a_bufs * a_bytes;
  int bsz = ((int)p.bblob.size() * 2 + 127) & ~127;
  p.smem_t = p.smem_b + bsz;
  p.smem_tw4 = p.smem_t;
  p.smem_bar = p.smem_tw4 + tw4_bytes;
#ifndef TCFFT_NO_ALIGN_SLACK
  p.smem_bytes = p.smem_bar + 64 + 1024;
#else
  p.smem_bytes = p.smem_bar + 64 /*mbarriers + TMEM address*/;
#endif
  int acols = p.st[0].tiles * (p.st[0].KP / 2);
  int dcols = 0;
  for (int s = 0; s < S; ++s) dcols = std::max(dcols, p.st[s].tiles * p.st[s].NP);
  int need = acols + dcols, tcols = 32;
  while (tcols < need) tcols <<= 1;
  if (tcols > 512) {
    if (err) *err = "TMEM budget exceeded";
    return false;
  }
  p.tmem_cols = tcols;
  p.tmem_a_cols = dcols;  // A region starts after D
  int by_tmem = 512 / tcols;
  int by_smem = 233472 / (p.smem_bytes + 1024);  // 228 KB per SM incl. 1 KB driver reserve per CTA
  p.ctas_per_sm = std::max(1, std::min(by_tmem, std::min(by_smem, 4)));
  // Pin occupancy: pad the shared-memory request so that no (ctas_per_sm+1)-th
  // CTA fits on an SM.  Otherwise an extra CTA (e.g. of the next grid under
  // programmatic dependent launch) lands beside ctas_per_sm TMEM holders and
  // spins in tcgen05.alloc, and its statically assigned chunks wait for a
  // whole neighbour's share: measured 1.8x slower four-step (round 1).
  // One CTA per SM: two warpgroups split every stage's tiles (kernel NWG).
  // TCFFT_NWG=<k> (experiment) asks for k warpgroups wherever tiles divide.
  {
    const char* e = experiment_env("TCFFT_NWG");
    int want = e ? std::atoi(e) : (p.ctas_per_sm == 1 ? 2 : 1);
    while (want > 1) {
      bool div = true;
      for (int s2 = 0; s2 < S; ++s2) div = div && (p.st[s2].tiles % want == 0);
      if (div) break;
      want /= 2;
    }
    p.nwg = std::max(1, want);
    // registers: 128 per thread at 512 threads per SM
    if (p.nwg > 1) p.ctas_per_sm = std::max(1, std::min(p.ctas_per_sm, 4 / p.nwg));
  }
  // Single-buffer passes (kernel ONEBUF): when the two-buffer layout leaves one
  // CTA per SM (chunks of 16384 elements), one buffer per chunk (staging ==
  // A operand == output staging) and a stage 1 run in two halves of tiles
  // (256 TMEM columns) fit two CTAs per SM; the SM's second CTA then hides
  // the load / MMA / barrier latencies the lone CTA exposed (1D 16384: 0.56 of
  // roofline with one CTA, round 1).  TCFFT_ONEBUF=0 (experiment) disables.
  {
    const char* e = experiment_env("TCFFT_ONEBUF");
    const bool allow = !e || std::atoi(e) != 0;
    const int dh = p.st[0].tiles / 2 * p.st[0].NP;
    const int a1 = p.st[0].tiles * (p.st[0].KP / 2);
    int dmax = 0;
    for (int s2 = 0; s2 < S; ++s2) dmax = std::max(dmax, p.st[s2].tiles * p.st[s2].NP);
    const int buf = (std::max(stage_bytes, a_bytes) + 1023) & ~1023;
    const int ob_bytes = buf + bsz + tw4_bytes + 64 + 1024;
    // (contiguous row inputs only: strided strip loads and the blocked rows of
    // the two-pass plans need the prefetch of the two-buffer layout, 2D 2048^2
    // 0.75 -> 0.63, two-pass 2^22 second pass 0.68 -> 0.57 of roofline
    // single-buffered, round 2)
    if (allow && kind == kPassRow && p.ctas_per_sm == 1 && E == 16384 && S >= 2 &&
        p.st[0].tiles % 2 == 0 && dh + a1 <= 256 &&
        dmax <= 256 && 2 * (ob_bytes + 1024) <= 233472) {
      p.onebuf = 1;
      p.nwg = 1;
      p.a_bufs = 1;
      p.smem_in = 0;
      p.smem_a = 0;
      p.a_bytes = buf;
      p.smem_b = buf;
      p.smem_t = p.smem_b + bsz;
      p.smem_tw4 = p.smem_t;
      p.smem_bar = p.smem_tw4 + tw4_bytes;
      p.smem_bytes = ob_bytes;
      p.tmem_cols = 256;
      p.tmem_a_cols = dh;
      p.ctas_per_sm = 2;
    }
  }
  const int pinned = ((233472 / (p.ctas_per_sm + 1) - 1024 + 1) + 127) & ~127;
  if (p.smem_bytes < pinned && p.ctas_per_sm * (pinned + 1024) <= 233472) p.smem_bytes = pinned;
  return true;
}

// Three-step 1D transform, N = N1 N2 N3 (each <= 256), n = N2 N3 n1 + N3 n2 + n3,
// k = k1 + N1 k2 + N1 N2 k3:
//   pass A: length-N1 FFTs over n1 (column strips of the [N1][N2 N3] input),
//           twiddle W_N^{(N3 n2 + n3) k1}, each column written as a contiguous
//           row: Y1[n2][n3][k1]
//   pass B: length-N2 FFTs over n2 (column strips of [N2][N3 N1], in place),
//           twiddle W_{N2 N3}^{n3 k2}: Y2[k2][n3][k1]
//   pass C: length-N3 FFTs over n3 (column strips of each [N3][N1] image k2),
//           stored straight into natural order X[k3][k2][k1] (4D tensor map)
// Every strided side moves C * 4 >= 64-byte runs per row: TMA strip copies with
// 16-byte runs reach ~60% of HBM bandwidth, 64-byte runs ~95%
// (tests/native/strip_io_probe.cu, round 1), so three passes of full-width
// traffic beat two passes of 16-byte runs (N1 = N2 = 2048) at these sizes.
static int build_three_step(Plan& plan, int nx, int lg, int64_t batch, std::string* err) {
  // N3 <= 256 (the 4D natural-order store of pass C); N1, N2 <= 4096 (2^36)
  int a = lg / 3, b = (lg - a) / 2, c = lg - a - b;
  if (c > 8) {
    c = 8;
    a = (lg - c) / 2;
    b = lg - c - a;
  }
  if (const char* e = experiment_env("TCFFT_THREE_SPLIT")) {  // experiment hook: "a,b,c" (log2 N1, N2, N3)
    int x, y, z;
    if (std::sscanf(e, "%d,%d,%d", &x, &y, &z) == 3 && x + y + z == lg) a = x, b = y, c = z;
  }
  const int N1 = 1 << a, N2 = 1 << b, N3 = 1 << c;
  PassPlan pa, pb, pc;
  if (!build_pass(pa, kPassStripT, N1, 0, batch, N2 * N3, err, nx)) return 6;
  if (!build_pass(pb, kPassStrip, N2, 0, batch, N3 * N1, err, (int64_t)N2 * N3, a)) return 6;
  if (!build_pass(pc, kPassStrip, N3, 0, batch * N2, N1, err)) return 6;
  if (pb.C > N1 || pc.C > N1 || pb.IMG != 1 || pc.IMG != 1) {
    if (err) *err = "unsupported three-step geometry";
    return 6;
  }
  // pass C output: X[b][k3][k2][k1] = 4D view {k1, k3 (stride N1 N2), k2 (stride N1), b (stride N)}
  pc.out.row_stride = (int64_t)N1 * N2;
  pc.out.img_split = N2;
  pc.out.img_stride = N1;
  pc.out.img_stride2 = nx;
  pa.ws_out = 1;
  pb.ws_in = pb.ws_out = 1;
  pc.ws_in = 1;
  plan.groups = 1;
  plan.group_bytes = (size_t)batch * (size_t)nx * 4;
  plan.ws_bytes = plan.group_bytes;
  plan.passes.push_back(std::move(pa));
  plan.passes.push_back(std::move(pb));
  plan.passes.push_back(std::move(pc));
  return 0;
}

// Two-pass 1D transform for 2^19 <= N <= 2^22, N = N1 N2 viewed as [N1][N2]
// (n = N2 n1 + n2, k = k1 + N1 k2):
//   pass 1: length-N1 FFTs down the columns (strips of C = E1/N1 columns,
//           C * 4 >= 32-byte runs), twiddle W_N^{n2 k1}; the chunk's staging
//           tile [k1][C] is stored CONTIGUOUSLY into the workspace, which
//           therefore holds Y[b][n2 / C][k1][n2 % C] (one flat store per chunk);
//   pass 2: length-N2 FFTs along k1-rows of that blocked array (one 4D box of
//           T rows x every block per chunk: C * T * 4-byte runs), transposed
//           store X[k1 + N1 k2] (T * 4 >= 32-byte runs).
// Each pass has exactly one strided side; the other side moves long runs, so
// the TMA engine's per-request cost is paid once per element instead of twice
// (three passes at >= 64-byte runs before, round 1).
static int build_two_pass_blocked(Plan& plan, int nx, int lg, int64_t batch, std::string* err) {
  const int a = lg / 2, b = lg - a;
  const int N1 = 1 << a, N2 = 1 << b;
  // pass 1: 8192-element strips (two CTAs per SM) for N1 >= 1024 — more
  // independent chunk chains per SM beat wider runs: 2^20 0.66 -> 0.74 of
  // roofline with 8 instead of 16 columns (round 2)
  // pass 2: 8192-element chunks for rows of <= 1024 (eight rows: 32-byte
  // output runs, two CTAs per SM; 2^20 0.73 -> 0.79), 16384 for 2048 (eight
  // rows; four rows would leave 16-byte runs: 0.29)
  const int E1 = N1 >= 1024 ? 8192 : std::min(16384, 16 * N1);
  const int E2 = N2 <= 1024 ? 8192 : std::min(16384, 16 * N2);
  PassPlan p1, p2;
  if (!build_pass(p1, kPassStrip, N1, 0, batch, N2, err, nx, 0, 0, E1)) return 6;
  if (p1.IMG != 1 || p1.C * 4 < 16) {
    if (err) *err = "unsupported two-pass geometry";
    return 6;
  }
  linear_io(p1.out, batch * (int64_t)nx, p1.E, p1.swz_out);
  if (!build_pass(p2, kPassRowTB, N2, batch * (int64_t)N1, batch, 0, err, 0, 0, p1.C, E2)) return 6;
  // pass 2 reads the tiles with their swizzle (T-row groups of a block are
  // whole swizzle atoms, aligned alike in the workspace and in shared memory)
  p2.in.swz = p2.swz_in = p1.swz_out;
  if (p1.swz_out && (p2.T * p1.C * 4) % (p1.C * 4 * 8) != 0) {
    if (err) *err = "two-pass: row group is not a whole swizzle atom";
    return 6;
  }
  p1.ws_out = 1;
  p2.ws_in = 1;
  plan.groups = 1;
  plan.group_bytes = (size_t)batch * (size_t)nx * 4;
  plan.ws_bytes = plan.group_bytes;
  plan.passes.push_back(std::move(p1));
  plan.passes.push_back(std::move(p2));
  return 0;
}

// Columns longer than one chunk (2D nx >= 8192), nx = N1 N2 viewed as
// [N1][N2][ny] (n = N2 n1 + n2, k = k1 + N1 k2), two column passes:
//   pass 2a: length-N1 FFTs over n1 (column strips of the [N1][N2 ny] image,
//            column c = n2 ny + y), twiddle W_nx^{n2 k1} = exponent
//            (c >> log2 ny) k1 -> workspace Y[b][k1][n2][y]
//   pass 2b: length-N2 FFTs over n2 (strips of each [N2][ny] image (b, k1)),
//            stored by a 4D tensor map {y, k2 (stride N1 ny), k1 (stride ny),
//            b (stride nx ny)} straight into X[b][k1 + N1 k2][y]
// (the three-step plan's passes B and C with a column dimension).
static int build_2d_split_columns(Plan& plan, int nx, int ny, int64_t batch, std::string* err) {
  int p = 0, q = 0;
  while ((1 << p) < nx) ++p;
  while ((1 << q) < ny) ++q;
  const int b2 = std::min(8, p - 5), b1 = p - b2;  // N2 = 256 (>= 16-column strips in pass 2b), N1 >= 32
  if (b1 > 12) {
    if (err) *err = "2D nx above 2^20 is not supported";
    return 6;
  }
  const int N1 = 1 << b1, N2 = 1 << b2;
  PassPlan pa, pb;
  if (!build_pass(pa, kPassStrip, N1, 0, batch, N2 * ny, err, nx, q)) return 6;
  if (!build_pass(pb, kPassStrip, N2, 0, batch * (int64_t)N1, ny, err)) return 6;
  if (pa.IMG != 1 || pb.IMG != 1) {
    if (err) *err = "2D nx >= 8192 needs ny >= " + std::to_string(pb.E / N2) + " (one column strip per chunk)";
    return 6;
  }
  if (pb.in.mode != kIoBox && pb.in.mode != kIoBoxR) {
    // one strip spans the whole row (C == ny): the flat view build_pass chose
    // cannot carry the 4D store, use the column box
    box_io(pb.in, batch * (int64_t)N1, N2, ny, pb.C);
    pb.out = pb.in;
    pb.swz_in = pb.swz_out = pb.in.swz;
    pb.flat = 0;
  }
  pb.out.row_stride = (int64_t)N1 * ny;
  pb.out.img_split = N1;
  pb.out.img_stride = ny;
  pb.out.img_stride2 = (int64_t)nx * ny;
  pa.ws_out = 1;
  pb.ws_in = 1;
  plan.ws_bytes = std::max<size_t>(plan.ws_bytes, (size_t)batch * (size_t)nx * (size_t)ny * 4);
  plan.passes.push_back(std::move(pa));
  plan.passes.push_back(std::move(pb));
  return 0;
}

int build_plan(Plan& plan, int dims, int nx, int ny, int64_t batch, std::string* err) {
  plan = Plan();
  plan.dims = dims;
  plan.nx = nx;
  plan.ny = ny;
  plan.batch = batch;
  auto pow2 = [](int n) { return n >= 2 && (n & (n - 1)) == 0; };
  if (!pow2(nx) || (dims == 2 && !pow2(ny))) {
    if (err) *err = "sizes must be powers of two >= 2";
    return 4;  // TCFFT_INVALID_SIZE
  }
  if (batch < 1) {
    if (err) *err = "batch must be >= 1";
    return 3;  // TCFFT_INVALID_VALUE
  }
  if (dims == 1 && nx <= 16384) {
    PassPlan p;
    if (!build_pass(p, kPassRow, nx, batch, 0, 0, err)) return 6;  // NOT_SUPPORTED
    plan.passes.push_back(std::move(p));
    return 0;
  }
  if (dims == 1) {
    // Four-step, N = N1 * N2 viewed as [N1][N2] (reference plan.py:35-44 chains
    // radix-8192 kernels instead; SPEC.md:452 leaves the schedule free):
    //   pass 1: length-N1 column FFTs, twiddle W_N^{n2 k1}, -> workspace
    //   pass 2: length-N2 row FFTs, transposed store X[k1 + N1 k2] -> output
    int lg = 0;
    while ((1 << lg) < nx) ++lg;
    if (lg > kMaxLog2_1D) {
      if (err) *err = "1D sizes above 2^" + std::to_string(kMaxLog2_1D) + " are not supported";
      return 6;
    }
    // Three passes for N >= 2^19 (every strided access keeps >= 64-byte
    // runs, see below); two passes up to 2^18, whose strips are >= 32 B wide.
    const char* eb = experiment_env("TCFFT_BLOCKED");
    if (lg >= 19 && lg <= 22 && (!eb || std::atoi(eb) != 0)) return build_two_pass_blocked(plan, nx, lg, batch, err);
    const char* e3 = experiment_env("TCFFT_THREE_PASS");
    if (lg >= 19 && (!e3 || std::atoi(e3) != 0)) return build_three_step(plan, nx, lg, batch, err);
    const int N1 = 1 << (lg / 2), N2 = 1 << (lg - lg / 2);
    // The batch is walked in L2-sized groups of G transforms (two launches per
    // group): the group's workspace (reused by every group) stays resident in
    // L2, so the intermediate never round-trips HBM and the 16-byte runs of
    // the transposed / strided accesses merge in L2 before write-back.
    // (opt-in: measured slower than one ungrouped launch per pass in round 1,
    // 17.9 vs 18.9 TFLOP/s for C3 at 128 MiB groups with CUDA-graph replay)
    int64_t group_mb = 0;
    if (const char* e = experiment_env("TCFFT_FOURSTEP_MB")) group_mb = std::max(0, std::atoi(e));
    int64_t G = batch;
    if (group_mb > 0) {
      G = std::max<int64_t>(1, (group_mb << 20) / ((int64_t)nx * 4));
      G = std::min<int64_t>(G, batch);
      while (batch % G) --G;
    }
    PassPlan p1, p2;
    if (!build_pass(p1, kPassStrip, N1, 0, G, N2, err, nx)) return 6;
    if (!build_pass(p2, kPassRowT, N2, G * (int64_t)N1, G, 0, err)) return 6;
    p1.ws_out = 1;
    p2.ws_in = 1;
    plan.groups = batch / G;
    plan.group_bytes = (size_t)G * (size_t)nx * 4;
    plan.ws_bytes = plan.group_bytes;
    plan.passes.push_back(std::move(p1));
    plan.passes.push_back(std::move(p2));
    return 0;
  }
  // 2D, row-major (nx, ny): contiguous rows (ny) first, then columns (nx)
  // at stride ny (reference executor.py:180-190).
  if (ny > 16384) {
    // rows longer than one chunk: the 1D multi-pass plan over batch * nx rows
    // (its last pass writes the output buffer)
    Plan rows;
    const int st = build_plan(rows, 1, ny, 0, batch * (int64_t)nx, err);
    if (st) return st;
    for (auto& q : rows.passes) plan.passes.push_back(std::move(q));
    plan.ws_bytes = rows.ws_bytes;
    if (rows.groups != 1) {
      if (err) *err = "2D rows: grouped row plans are not supported";
      return 6;
    }
  } else {
    PassPlan rowp;
    if (!build_pass(rowp, kPassRow, ny, batch * (int64_t)nx, 0, 0, err)) return 6;
    plan.passes.push_back(std::move(rowp));
  }
  if (nx <= 4096) {
    PassPlan colp;
    if (!build_pass(colp, kPassStrip, nx, 0, batch, ny, err)) return 6;
    plan.passes.push_back(std::move(colp));
    return 0;
  }
  return build_2d_split_columns(plan, nx, ny, batch, err);
}

// Distributed single 1D transform over `world` ranks,
// N = N1 N2 viewed as [N1][N2] (n = N2 n1 + n2, k = k1 + N1 k2), G = world:
//   rank g input : the column slab x[N2 n1 + n2], n2 in [g N2/G, (g+1) N2/G),
//                  stored [N1][N2/G]
//   pass 0       : length-N1 column FFTs of the slab, twiddle W_N^{n2 k1}
//                  (global n2 = g N2/G + column: tw4_col0), in place
//   exchange     : all-to-all of the N1/G-row blocks (NCCL), then the received
//                  [G][N1/G][N2/G] blocks are unpacked into rows [N1/G][N2]
//                  (tcfftDistUnpack: G strided device copies)
//   pass 1       : length-N2 row FFTs, transposed store: rank g output
//                  [N2][N1/G] = X[k1 + N1 k2] for k1 in [g N1/G, (g+1) N1/G)
// Both passes are the single-GPU four-step kernels; N1, N2 <= 4096 (N <= 2^24).
int build_plan_dist(Plan& plan, int nx, int rank, int world, std::string* err, bool fused) {
  plan = Plan();
  plan.dims = 1;
  plan.nx = nx;
  plan.batch = 1;
  auto pow2 = [](int n) { return n >= 1 && (n & (n - 1)) == 0; };
  if (nx < 2 || !pow2(nx)) {
    if (err) *err = "sizes must be powers of two >= 2";
    return 4;
  }
  if (!pow2(world) || rank < 0 || rank >= world) {
    if (err) *err = "world must be a power of two and 0 <= rank < world";
    return 3;
  }
  int lg = 0;
  while ((1 << lg) < nx) ++lg;
  const int a = lg / 2, b = lg - a;
  const int N1 = 1 << a, N2 = 1 << b;
  if (N1 > 4096 || N2 > 4096 || N1 % world || N2 % world) {
    if (err) *err = "distributed transforms need N1, N2 <= 4096 divisible by the world size";
    return 6;
  }
  const int cols = N2 / world, rows = N1 / world;
  PassPlan p0, p1;
  // (fused: the wide strips of the single-GPU two-pass plan, >= 32-byte runs)
  const int E1 = fused ? std::min(16384, 16 * N1) : 0;
  if (!build_pass(p0, kPassStrip, N1, 0, 1, cols, err, nx, 0, 0, E1)) return 6;
  if (p0.IMG != 1 || cols % p0.C) {
    if (err) *err = "distributed transform: column slab narrower than one strip";
    return 6;
  }
  p0.tw4_col0 = (int64_t)rank * cols;
  if (fused) {
    // Pass 0's staging tile [k1][C] (N1 rows) splits into `world` slices of
    // N1/world rows; slice h goes byte for byte to rank h's receive buffer at
    // global column block (rank cols + chunk C) / C, so every rank receives
    // R[n2 / C][k1 local][n2 % C]: the blocked layout of the single-GPU
    // two-pass plan, read by the blocked-rows pass (kPassRowTB).
    const int C = p0.C;
    const int slice = rows * C * 4;
    if (rows % 8 || slice % 256 || N2 / C > 256) {
      if (err) *err = "fused distributed transform: unsupported slice geometry";
      return 6;
    }
    p0.out.mode = kIoPeer;
    p0.out.n_sub = world;
    p0.out.sub_bytes = slice;
    p0.out.npeer = world;
    p0.out.peer_blk0 = (int64_t)rank * (cols / C);
    // (p0.out.swz keeps the strip's swizzle: the slices are stored verbatim)
    const int E2 = std::min(16384, 16 * N2);
    if (!build_pass(p1, kPassRowTB, N2, rows, 1, 0, err, 0, 0, C, E2)) return 6;
    p1.in.swz = p1.swz_in = p0.swz_out;
    if ((p1.T * C * 4) % (C * 4 * 8) != 0) {
      if (err) *err = "fused distributed transform: row group is not a whole swizzle atom";
      return 6;
    }
  } else {
    if (!build_pass(p1, kPassRowT, N2, rows, 1, 0, err)) return 6;
  }
  plan.passes.push_back(std::move(p0));
  plan.passes.push_back(std::move(p1));
  plan.dist = fused ? 2 : 1;
  return 0;
}

}  // namespace tcfft
