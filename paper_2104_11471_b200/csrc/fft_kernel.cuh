// fft_kernel.cuh - one persistent sm_100a kernel per HBM pass of the batched
// FP16 C2C FFT.
//
// Per CTA (128 threads; thread t <-> TMEM lane t <-> MMA row t):
//   TMA tensor load of a chunk (E complex fp16 = 4E bytes, 128B-swizzled) ->
//   stage 1 : each thread gathers the R_1 inputs of its butterfly(s) from the
//             natural-order staging buffer (digit reversal folded into the
//             addresses) and writes them to TMEM as the A operand;
//             tcgen05.mma (A from TMEM, B = real 2R x 2R DFT block matrix in
//             SMEM, D fp32 in TMEM)
//   stage s>1: the previous epilogue wrote this stage's A operand into SMEM in
//             the UMMA MN-major layout (split re/im planes, 16B vector stores);
//             tcgen05.mma (A, B from SMEM)
//   epilogue: tcgen05.ld the accumulator row, apply the NEXT stage's twiddle in
//             fp32 (packed FFMA2; the per-row twiddle sequence c*w^j comes from
//             a register recurrence, no table traffic), round once to fp16
//             (cvt.rn.f16x2) and store the next operand, or (last stage) the
//             natural-order output staging tile, which a TMA tensor store
//             writes back to HBM.
// HBM is touched exactly once per element per pass.  See DESIGN.md.
#pragma once
#include <cuda.h>
#include <cstdint>
#include <type_traits>
#include "sm100.cuh"
#include "plan.hpp"

namespace tcfft {

// One side (load or store) of a pass, see plan.hpp IoDesc.
struct KIo {
  int32_t mode;         // IoMode
  int32_t box_rows, n_sub, sub_bytes, chunk_rows;
  int32_t C, spi;       // box: columns per chunk, chunks per image
  int32_t isplit;       // box: 4D map, image index = outer * isplit + inner (0: 3D)
  int32_t pitch_bytes;  // pitch mode: staging pitch per transform
  int64_t gstride_bytes;  // pitch mode: global distance between transforms (batch_stride * 4)
  int64_t count;        // pitch mode: transforms in the pass
  const uint8_t* gptr;  // pitch mode: raw global pointer, set per execution
  int32_t npeer;        // peer mode: slices / ranks
  int64_t peer_blk0;    // peer mode: global column block of chunk 0
  const uint8_t* peers[8];  // peer mode: every rank's receive buffer (peer / IPC-mapped device pointers)
};

struct KParams {
  int64_t chunks;
  int32_t T;  // transforms per chunk
  int32_t gstride, ostride, swz_in, swz_out;
  int32_t tiles_max;
  KIo in, out;
  const RowInfo* rows_tab;
  const uint16_t* bblob;
  int32_t bbytes;
  int32_t smem_a, a_stride, smem_b, smem_bar, smem_tw4;
  int64_t tw4_total;  // four-step pass 1: full transform length
  int32_t tw4_shift;  // exponent uses (column >> tw4_shift) (three-step pass B)
  int64_t tw4_col0;   // global column of the pass's column 0 (distributed plans)
  int32_t tw4_nk;     // number of final-stage k values (N1 / R_S)
  int32_t tw4_s;      // N1 / R_S
  int32_t late_wait;     // wait for the previous store's shared-memory read after issuing stage 1
  int32_t gather_ahead;  // gather chunk i+1 while chunk i's last MMAs run
  int32_t pipe;          // software-pipelined chunk loop (else the simple lock-step loop)
  int32_t pdl;           // PDL trigger point: 1 = last chunk, 2 = CTA start
  unsigned long long* trace;  // TCFFT_TRACE builds: per-CTA globaltimer stamps
  unsigned long long* ctr;    // dynamic chunk tickets {next, retired CTAs}; null = static
  int64_t static_chunks;      // with ctr: chunks [0, static_chunks) are statically striped
};

namespace dev {

using namespace sm100;

// ---------------------------------------------------------------- compile-time pass geometry
// kModeStrip4: column strips in, 4D tensor-map store out (three-step pass C)
// kModeRowU: rows of 4 .. 16 whose batch is not a multiple of 32 elements
// (unswizzled [total/4][4] staging)
// kModeRowTB: rows of a blocked array in (runtime gather addressing), transposed out
enum : int { kModeRow = 0, kModeStrip = 1, kModeRowT = 2, kModeStrip4 = 3, kModeRowU = 5, kModeRowTB = 6 };

template <int E_, int R1_, int R2_, int R3_, int MODE_>
struct Cfg {
  static constexpr int E = E_;
  static constexpr bool ROW_IN = MODE_ == kModeRow || MODE_ == kModeRowT || MODE_ == kModeRowU;  // contiguous rows in
  static constexpr bool ROW = MODE_ == kModeRow || MODE_ == kModeRowU;  // ... and contiguous rows out
  static constexpr int S = (R2_ == 0) ? 1 : ((R3_ == 0) ? 2 : 3);
  static constexpr int N = R1_ * (R2_ ? R2_ : 1) * (R3_ ? R3_ : 1);
  __host__ __device__ static constexpr int R(int s) { return s == 0 ? R1_ : (s == 1 ? R2_ : R3_); }
  static constexpr int RL = R(S - 1);
  // radix-64 first stages gather their TMEM A operand in planar K order
  // (re_0..re_63, im_0..im_63) so that their B matrix equals the planar one of
  // a following radix-64 stage (shared: 32 KB of SMEM saved); plan.cpp mirrors
  static constexpr bool PLANAR0 = R1_ == 64;
  __host__ __device__ static constexpr int KP(int s) { return 2 * R(s) < 16 ? 16 : 2 * R(s); }
  __host__ __device__ static constexpr int NP(int s) { return KP(s); }
  __host__ __device__ static constexpr int T(int s) { return E / (128 * R(s)); }
  __host__ __device__ static constexpr int SBO(int s) { return 32 * R(s) + 16; }  // padded: consecutive 8-row groups hit distinct banks
  __host__ __device__ static constexpr int TILEB(int s) { return 16 * SBO(s); }
  // B matrices: stage 0 (interleaved K), then one planar-K matrix per distinct
  // radix run (stages s >= 2 with R(s) == R(s-1) share the previous matrix;
  // TCFFT_NO_BDEDUPE builds keep one copy per stage)
  __host__ __device__ static constexpr int BSZ(int s) { return KP(s) * NP(s) * 2; }
#ifdef TCFFT_NO_BDEDUPE
  __host__ __device__ static constexpr bool BSHARE(int s) { return false; }
#else
  __host__ __device__ static constexpr bool BSHARE(int s) {
    return (s >= 2 && R(s) == R(s - 1)) || (s == 1 && PLANAR0 && R(1) == R(0));
  }
#endif
  __host__ __device__ static constexpr int BOFF(int s) {
    return s == 0 ? 0 : (BSHARE(s) ? BOFF(s - 1) : BOFF(s - 1) + (BSHARE(s - 1) ? 0 : BSZ(s - 1)));
  }
  // writer row-block interleave, plan.cpp writer_groups()
  __host__ __device__ static constexpr int HSTEP(int s) {
    return (R(s) == 32 && E / R(s + 1) >= 8 * R(s)
                ? 8
                : (R(s) <= 32 ? 128 / R(s) : (E / R(s + 1) >= 8 * R(s) ? 8 : (E / R(s + 1) >= 4 * R(s) ? 4 : 2)))) *
           SBO(s + 1);
  }
  __host__ __device__ static constexpr int IMOFF(int s) { return 16 * R(s + 1); }
  __host__ __device__ static constexpr int tmax(int a, int b) { return a > b ? a : b; }
  static constexpr int TMAX = tmax(T(0), tmax(T(S > 1 ? 1 : 0), T(S - 1)));
  // staging strides (words) and swizzle, compile-time for contiguous row passes
  static constexpr int GS = N / R(0);
  static constexpr int OS = N / RL;
  // row passes: 128B-swizzled staging for N == 32 and N >= 2048; 64 <= N <= 1024
  // use padded per-transform staging (plan.cpp pitch_mode) without swizzle
  // Rows of 64 .. 256 in 4096-element chunks go through the flat 128B-swizzled
  // map (one TMA box per chunk instead of 16 .. 64 per-row bulk copies: 1D 256
  // 0.82 -> 0.86 of roofline despite 2-/4-way conflicted gathers / stores);
  // the small-batch 2048-element chunks (C1) keep the padded pitch (-3% flat).
  static constexpr bool PITCH = ROW_IN && N >= 64 && N <= 1024 && !(N <= 256 && E_ == 4096);
  // (rows of 4 .. 16 too: each lane owns one whole transform, and the swizzle
  // spreads the lanes' N-word strides over the banks: 16-way -> 2-way at N = 16)
  static constexpr uint32_t SWZ = (N >= 4 && !PITCH && MODE_ != kModeRowU) ? 0x70u : 0u;
  static constexpr bool AFF_IN = ROW_IN && (SWZ == 0 || (GS * 4) % 1024 == 0);
  static constexpr bool AFF_OUT = ROW && (SWZ == 0 || (OS * 4) % 1024 == 0);
  // TMEM: D region (max over stages) then the stage-1 A region
  __host__ __device__ static constexpr int DC(int s) { return T(s) * NP(s); }
  static constexpr int DCOLS = tmax(DC(0), tmax(DC(S > 1 ? 1 : 0), DC(S - 1)));
  static constexpr int ACOLS = T(0) * KP(0) / 2;
  static constexpr int NEED = DCOLS + ACOLS;
  static constexpr uint32_t COLS = NEED <= 32 ? 32 : NEED <= 64 ? 64 : NEED <= 128 ? 128 : NEED <= 256 ? 256 : 512;
  static_assert(NEED <= 512, "TMEM budget");
};

DEVI uint32_t swz(uint32_t byte, uint32_t mask) { return byte ^ ((byte >> 3) & mask); }

DEVI void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
DEVI void sts32(uint32_t a, uint32_t x) { asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(x) : "memory"); }
DEVI uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}

// Load NP fp32 accumulator columns of this thread's row.
template <int NP>
DEVI void load_acc(uint32_t taddr, float* x) {
  uint32_t* r = reinterpret_cast<uint32_t*>(x);
  if constexpr (NP == 16) {
    tmem_ld16(taddr, r);
  } else if constexpr (NP == 32) {
    tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(r));
  } else {
    static_assert(NP == 64, "NP");
    tmem_ld32(taddr, *reinterpret_cast<uint32_t(*)[32]>(r));
    tmem_ld32(taddr + 32, *reinterpret_cast<uint32_t(*)[32]>(r + 32));
  }
  tmem_wait_ld();
}

// Load K consecutive 32-bit TMEM columns of this thread's lane (no wait).
template <int K>
DEVI void tmem_ld_words(uint32_t taddr, uint32_t* r) {
  if constexpr (K >= 8) {
    tmem_ld8(taddr, r);
    tmem_ld_words<K - 8>(taddr + 8, r + 8);
  } else if constexpr (K >= 4) {
    tmem_ld4(taddr, r);
    tmem_ld_words<K - 4>(taddr + 4, r + 4);
  } else if constexpr (K >= 2) {
    tmem_ld2(taddr, r);
    tmem_ld_words<K - 2>(taddr + 2, r + 2);
  } else if constexpr (K == 1) {
    tmem_ld1(taddr, r);
  }
}

// Per-thread row records (host-built RowInfo fields) kept in spare TMEM
// columns instead of registers: [stage-1 gather bases | per writer stage and
// tile: addr, w (, c) | per final tile: addr (, k, c, w)].
template <class C, bool TW4>
struct Rec {
  __host__ __device__ static constexpr int WS(int s) { return s == 0 ? 3 : 5; }
  static constexpr int FW = TW4 ? 6 : 1;
  __host__ __device__ static constexpr int OFF_W(int s) { return s == 0 ? C::T(0) : OFF_W(s - 1) + C::T(s - 1) * WS(s - 1); }
  static constexpr int OFF_F = OFF_W(C::S - 1);
  static constexpr int N = OFF_F + C::T(C::S - 1) * FW;
  static constexpr int COL = C::DCOLS + C::ACOLS;
#ifndef TCFFT_TMEMREC
  static constexpr bool IN_TMEM = false;
#else
  static constexpr bool IN_TMEM = COL + N <= (int)C::COLS;
#endif
};

DEVI float2 neg2(float2 a) { return make_float2(-a.x, -a.y); }  // folded into FFMA2 operand negation

// Stage 1: gather R inputs (natural order) into TMEM A (interleaved re/im K order).
template <class C>
DEVI void gather_to_tmem(uint32_t s_in, int gbase, int gstride, uint32_t swzmask, uint32_t taddr) {
  constexpr int R = C::R(0);
  constexpr int KC = C::KP(0) / 2;  // TMEM columns (2 fp16 per column)
  uint32_t v[KC];
  if constexpr (C::AFF_IN) {
    const uint32_t b0 = s_in + swz((uint32_t)gbase * 4u, C::SWZ);
#pragma unroll
    for (int m = 0; m < KC; ++m) v[m] = (m < R) ? lds32(b0 + m * C::GS * 4) : 0u;
  } else {
    const int gs = C::ROW_IN ? C::GS : gstride;
    const uint32_t msk = C::ROW_IN ? C::SWZ : swzmask;
#pragma unroll
    for (int m = 0; m < KC; ++m)
      v[m] = (m < R) ? lds32(s_in + swz((uint32_t)(gbase + m * gs) * 4u, msk)) : 0u;
  }
  if constexpr (C::PLANAR0) {
    // v[m] = (re_m | im_m << 16): column c < KC/2 holds (re_2c, re_2c+1),
    // column KC/2 + c holds (im_2c, im_2c+1)
    uint32_t w[KC];
#pragma unroll
    for (int c = 0; c < KC / 2; ++c) {
      w[c] = __byte_perm(v[2 * c], v[2 * c + 1], 0x5410);
      w[KC / 2 + c] = __byte_perm(v[2 * c], v[2 * c + 1], 0x7632);
    }
#pragma unroll
    for (int q = 0; q < KC / 16; ++q) tmem_st16(taddr + 16 * q, w + 16 * q);
  } else if constexpr (KC == 8) {
    tmem_st8(taddr, v);
  } else if constexpr (KC == 16) {
    tmem_st16(taddr, v);
  } else {
    static_assert(KC == 32 || KC == 64, "KC");
#pragma unroll
    for (int q = 0; q < KC / 16; ++q) tmem_st16(taddr + 16 * q, v + 16 * q);
  }
}

// Accumulator row of stage s, outputs [j0, j0 + G): re -> xr[], im -> xi[].
// D columns are planar: re_j at column j, im_j at column R + j.
template <int R, int G>
DEVI void load_group(uint32_t taddr, int j0, float* xr, float* xi) {
  if constexpr (R <= 8) {
    uint32_t r[16];
    tmem_ld16(taddr, r);  // NP = 16: re 0..R-1, im R..2R-1
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < G; ++j) {
      xr[j] = __uint_as_float(r[j]);
      xi[j] = __uint_as_float(r[R + j]);
    }
  } else {
    static_assert(G == 16, "G");
    tmem_ld16(taddr + j0, reinterpret_cast<uint32_t*>(xr));
    tmem_ld16(taddr + R + j0, reinterpret_cast<uint32_t*>(xi));
    tmem_wait_ld();
  }
}

// Twiddle sequence t_j = c * w^j, advanced two outputs at a time (packed
// FFMA2 on the pairs (t_j, t_{j+1})); exact values come from the host / the
// per-chunk table, the recurrence adds ~R ulps of fp32 error.
struct TwSeq {
  float2 tr, ti, w2r, w2i;
  DEVI TwSeq(float2 c, float2 w) {
    const float2 w2 = make_float2(w.x * w.x - w.y * w.y, 2.f * w.x * w.y);
    w2r = make_float2(w2.x, w2.x);
    w2i = make_float2(w2.y, w2.y);
    tr = make_float2(c.x, c.x * w.x - c.y * w.y);
    ti = make_float2(c.y, c.x * w.y + c.y * w.x);
  }
  // y = x * t for the current pair, then advance
  DEVI void apply(float2 xr, float2 xi, float2& yr, float2& yi) {
    yr = ffma2(neg2(xi), ti, fmul2(xr, tr));  // xr*tr - xi*ti
    yi = ffma2(xi, tr, fmul2(xr, ti));        // xr*ti + xi*tr
    const float2 ntr = ffma2(neg2(ti), w2i, fmul2(tr, w2r));
    const float2 nti = ffma2(ti, w2r, fmul2(tr, w2i));
    tr = ntr;
    ti = nti;
  }
};

// Writer epilogue of stage s: y_j = x_j * c * w^j (fp32, packed pairs),
// rounded once to fp16 split planes, 16B stores into stage s+1's MN-major A.
// Processed in groups of (up to) 16 outputs to bound register pressure.
template <class C, int s>
DEVI void writer_epilogue(uint32_t taddr, uint32_t dst, float2 c, float2 w) {
  constexpr int R = C::R(s);
  constexpr int G = R < 16 ? R : 16;
  TwSeq tw(c, w);
#pragma unroll
  for (int g = 0; g < R / G; ++g) {
    float xr[G], xi[G];
    load_group<R, G>(taddr, g * G, xr, xi);
#pragma unroll
    for (int h = 0; h < G / 8; ++h) {
      uint32_t pr[4], pi[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = 8 * h + 2 * q;
        float2 yr, yi;
        tw.apply(make_float2(xr[j], xr[j + 1]), make_float2(xi[j], xi[j + 1]), yr, yi);
        pr[q] = pack_half2(yr.x, yr.y);
        pi[q] = pack_half2(yi.x, yi.y);
      }
      const uint32_t d = dst + ((g * G) / 8 + h) * C::HSTEP(s);
      sts128(d, pr[0], pr[1], pr[2], pr[3]);
      sts128(d + C::IMOFF(s), pi[0], pi[1], pi[2], pi[3]);
    }
  }
}

// Final epilogue: natural-order interleaved output into the staging tile,
// optionally times the four-step twiddle c4 * w4^j.
template <class C, bool TW4>
DEVI void final_epilogue(uint32_t taddr, uint32_t s_out, int obase, int ostride, uint32_t swzmask, float2 c4,
                         float2 w4) {
  constexpr int R = C::RL;
  constexpr int G = R < 16 ? R : 16;
  const int os = C::ROW ? C::OS : ostride;
  const uint32_t msk = C::ROW ? C::SWZ : swzmask;
  const uint32_t b0 = s_out + swz((uint32_t)obase * 4u, C::SWZ);
  TwSeq tw(c4, w4);
#pragma unroll
  for (int g = 0; g < R / G; ++g) {
    float xr[G], xi[G];
    load_group<R, G>(taddr, g * G, xr, xi);
#pragma unroll
    for (int jp = 0; jp < G / 2; ++jp) {
      float2 yr = make_float2(xr[2 * jp], xr[2 * jp + 1]);
      float2 yi = make_float2(xi[2 * jp], xi[2 * jp + 1]);
      if constexpr (TW4) tw.apply(make_float2(xr[2 * jp], xr[2 * jp + 1]), make_float2(xi[2 * jp], xi[2 * jp + 1]), yr, yi);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int j = g * G + 2 * jp + e;
        const uint32_t wv = e ? pack_half2(yr.y, yi.y) : pack_half2(yr.x, yi.x);
        if constexpr (C::AFF_OUT)
          sts32(b0 + j * C::OS * 4, wv);
        else
          sts32(s_out + swz((uint32_t)(obase + j * os) * 4u, msk), wv);
      }
    }
  }
}

// I/O modes a kernel MODE can meet (plan.cpp build_pass / the exec paths):
// the branches of the others compile out of thread 0's load / store issue,
// which sits on every chunk's critical path (two extra runtime branches there
// measured -5% on C3, profiles/exp_views2d_r02.txt; these sets +2%,
// profiles/exp_ioset_r02.txt)
template <int MODE, bool TW4>
struct IoSet {
  static constexpr uint32_t ROWS = (1u << kIoPitch) | (1u << kIoFlat) | (1u << kIoFlat3) | (1u << kIoRank1);
  static constexpr uint32_t BOXES = (1u << kIoBox) | (1u << kIoBoxR);
  static constexpr bool ROWK = MODE == kModeRow || MODE == kModeRowU;
  // (column strips load boxes or flat tiles: never per-transform pitch copies or blocked rows)
  static constexpr uint32_t STRIP_IN = ~((1u << kIoPitch) | (1u << kIoBlk));
  static constexpr uint32_t IN = MODE == kModeRowTB ? (1u << kIoBlk) : (ROWK || MODE == kModeRowT) ? ROWS : STRIP_IN;
  // stores: untwiddled column strips write where they read (2D columns), the
  // 4D natural-order strips (three-step pass C, 2D split columns) one box;
  // twiddled strips meet every store mode (contiguous / peer tiles, pitch rows)
  static constexpr uint32_t OUT = (MODE == kModeRowTB || MODE == kModeRowT) ? BOXES
                                  : ROWK                                   ? ROWS
                                  : MODE == kModeStrip4                    ? (1u << kIoBox)
                                  : (MODE == kModeStrip && !TW4)
                                      ? BOXES | (1u << kIoFlat) | (1u << kIoFlat3) | (1u << kIoRank1)
                                      : ~0u;
};
// io.mode == M, decided at compile time when SET excludes M or holds only M
template <uint32_t SET, int M>
DEVI bool io_is(const KIo& io) {
  if constexpr (!((SET >> M) & 1u)) return false;
  else if constexpr (SET == (1u << M)) return true;
  else return io.mode == M;
}

// chunk ids fit 32 bits (< 2^32 chunks of >= 1024 elements): 32-bit instead of
// 64-bit division on thread 0's per-chunk issue path
DEVI uint32_t chunk32(int64_t c) { return (uint32_t)c; }

template <uint32_t SET>
DEVI void issue_load(const CUtensorMap* tm, const KIo& io, int T, int64_t chunk, uint8_t* dst, uint64_t* bar) {
  if (io_is<SET, kIoPitch>(io)) {
    const int64_t t0 = chunk * T;
    const int nt = (int)min((int64_t)T, io.count - t0);
    mbar_arrive_expect_tx(bar, (uint32_t)(nt * io.sub_bytes));
    for (int i = 0; i < nt; ++i)
      bulk_g2s(dst + i * io.pitch_bytes, io.gptr + (t0 + i) * io.gstride_bytes, io.sub_bytes, bar);
    return;
  }
  mbar_arrive_expect_tx(bar, (uint32_t)(io.n_sub * io.sub_bytes));
  if (io_is<SET, kIoFlat3>(io)) {  // whole > 256-row flat chunk in one 3D box
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(0), "r"(0), "r"((int32_t)(chunk * io.n_sub)), "r"(smem_u32(bar))
        : "memory");
  } else if (io_is<SET, kIoBlk>(io)) {  // C-row group rb of every Bw-wide block of one image, 4D boxes of <= 256 blocks
    const int32_t img = (int32_t)(chunk32(chunk) / (uint32_t)io.spi), rb = (int32_t)(chunk32(chunk) % (uint32_t)io.spi);
    const int32_t bpb = io.box_rows;  // blocks per box
    for (int i = 0; i < io.n_sub; ++i)
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
          "%5}], [%6];" ::"r"(smem_u32(dst + i * io.sub_bytes)),
          "l"(tm), "r"(0), "r"(rb), "r"(i * bpb), "r"(img), "r"(smem_u32(bar))
          : "memory");
  } else if (io_is<SET, kIoBoxR>(io)) {  // whole > 256-row strip in one 4D box
    const int32_t img = (int32_t)(chunk32(chunk) / (uint32_t)io.spi), cb = (int32_t)(chunk32(chunk) % (uint32_t)io.spi);
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(tm), "r"(cb * io.C), "r"(0), "r"(0), "r"(img), "r"(smem_u32(bar))
        : "memory");
  } else if (io_is<SET, kIoRank1>(io)) {
    const int32_t e0 = (int32_t)(chunk * io.chunk_rows);
    for (int i = 0; i < io.n_sub; ++i) tma_load_1d(dst + i * io.sub_bytes, tm, e0 + i * io.box_rows, bar);
  } else if (io_is<SET, kIoFlat>(io)) {
    const int32_t row0 = (int32_t)(chunk * io.chunk_rows);
    for (int i = 0; i < io.n_sub; ++i) tma_load_2d(dst + i * io.sub_bytes, tm, 0, row0 + i * io.box_rows, bar);
  } else {
    const int32_t img = (int32_t)(chunk32(chunk) / (uint32_t)io.spi), cb = (int32_t)(chunk32(chunk) % (uint32_t)io.spi);
    for (int i = 0; i < io.n_sub; ++i) {
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4}], [%5];" ::"r"(smem_u32(dst + i * io.sub_bytes)),
            "l"(tm), "r"(cb * io.C), "r"(i * io.box_rows), "r"(img), "r"(smem_u32(bar))
            : "memory");
    }
  }
}

template <uint32_t SET, bool D4 = false>
DEVI void issue_store(const CUtensorMap* tm, const KIo& io, int T, int64_t chunk, const uint8_t* src) {
  if (io_is<SET, kIoPitch>(io)) {
    const int64_t t0 = chunk * T;
    const int nt = (int)min((int64_t)T, io.count - t0);
    for (int i = 0; i < nt; ++i)
      bulk_s2g(const_cast<uint8_t*>(io.gptr) + (t0 + i) * io.gstride_bytes, src + i * io.pitch_bytes, io.sub_bytes);
  } else if (io_is<SET, kIoLinear>(io)) {  // the staging tile byte for byte, one bulk copy
    bulk_s2g(const_cast<uint8_t*>(io.gptr) + chunk * (int64_t)io.sub_bytes, src, io.sub_bytes);
  } else if (io_is<SET, kIoPeer>(io)) {
    // distributed plans: row slice h of the tile straight into rank h's
    // receive buffer (over NVLink for a peer GPU), at this chunk's global
    // column block: the exchange is the pass's own store
    const int64_t blk = io.peer_blk0 + chunk;
    for (int h = 0; h < io.npeer; ++h)
      bulk_s2g(const_cast<uint8_t*>(io.peers[h]) + blk * io.sub_bytes, src + h * io.sub_bytes, io.sub_bytes);
  } else if (io_is<SET, kIoFlat3>(io)) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(tm),
                 "r"(0), "r"(0), "r"((int32_t)(chunk * io.n_sub)), "r"(smem_u32(src))
                 : "memory");
  } else if (io_is<SET, kIoBoxR>(io)) {
    const int32_t img = (int32_t)(chunk32(chunk) / (uint32_t)io.spi), cb = (int32_t)(chunk32(chunk) % (uint32_t)io.spi);
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(tm),
                 "r"(cb * io.C), "r"(0), "r"(0), "r"(img), "r"(smem_u32(src))
                 : "memory");
  } else if (io_is<SET, kIoRank1>(io)) {
    const int32_t e0 = (int32_t)(chunk * io.chunk_rows);
    for (int i = 0; i < io.n_sub; ++i) tma_store_1d(tm, e0 + i * io.box_rows, src + i * io.sub_bytes);
  } else if (io_is<SET, kIoFlat>(io)) {
    const int32_t row0 = (int32_t)(chunk * io.chunk_rows);
    for (int i = 0; i < io.n_sub; ++i) tma_store_2d(tm, 0, row0 + i * io.box_rows, src + i * io.sub_bytes);
  } else {
    const int32_t img = (int32_t)(chunk32(chunk) / (uint32_t)io.spi), cb = (int32_t)(chunk32(chunk) % (uint32_t)io.spi);
    for (int i = 0; i < io.n_sub; ++i) {
      if constexpr (D4)
        asm volatile(
            "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(tm),
            "r"(cb * io.C), "r"(i * io.box_rows), "r"(img % io.isplit), "r"(img / io.isplit),
            "r"(smem_u32(src + i * io.sub_bytes))
            : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(tm),
            "r"(cb * io.C), "r"(i * io.box_rows), "r"(img), "r"(smem_u32(src + i * io.sub_bytes))
            : "memory");
    }
  }
  bulk_commit();
}

// Issue the MMAs of stage s (one elected thread).  Stage 0 may be issued for
// a tile range [TB, TE) whose accumulators start at TMEM column (t - TB) * NP
// (single-buffer passes run stage 0 in two halves sharing one D region).
template <class C, int s, int TB = 0, int TE = C::T(s), bool DSHIFT = false>
DEVI void issue_stage_mma(uint32_t s_a, uint32_t s_b, uint32_t tD, uint32_t tA) {
  constexpr int KP = C::KP(s), NP = C::NP(s), T = C::T(s);
  if constexpr (s == 0) {
    constexpr uint32_t idesc = make_idesc_f16(128, NP, 0, 0);  // A (TMEM) K-major, B K-major
#pragma unroll
    for (int t = TB; t < TE; ++t)
#pragma unroll
      for (int q = 0; q < KP / 16; ++q)
        mma_ts(tD + (DSHIFT ? t - TB : t) * NP, tA + t * (KP / 2) + q * 8,
               make_sdesc(s_b + C::BOFF(s) + q * 32 * NP, 128, 256), idesc, q > 0);
  } else {
    constexpr uint32_t idesc = make_idesc_f16(128, NP, 1, 0);  // A MN-major (split planes), B K-major
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
      for (int q = 0; q < KP / 16; ++q)
        mma_ss(tD + t * NP, make_sdesc(s_a + t * C::TILEB(s) + q * 256, 128, C::SBO(s)),
               make_sdesc(s_b + C::BOFF(s) + q * 32 * NP, 128, 256), idesc, q > 0);
  }
}

}  // namespace dev

// NWG warpgroups of 128 threads: warpgroup w handles tiles t = w, w + NWG, ...
// of every stage (TMEM lane quarter = warp % 4).  Two warpgroups for the
// one-CTA-per-SM passes (E = 16384), whose chunk loop is otherwise latency
// bound on a single warp per SM sub-partition.
// ONEBUF: single-buffer passes (chunks of 16384 elements, two CTAs per SM).
// One shared-memory buffer holds a chunk for its whole life: TMA load ->
// stage-1 gather (to TMEM) -> every later stage's A operand -> output staging
// -> TMA store; the next chunk's load is issued once the store has read the
// buffer, while the SM's other CTA computes.  Stage 1 runs in two halves of
// tiles sharing one accumulator region, so a CTA needs 256 TMEM columns
// (D/2 + the stage-1 A operand, then the full D of later stages over the dead
// A operand) and two CTAs fit an SM.
template <int E, int R1, int R2, int R3, int MINB, int MODE, bool TW4, int NWG = 1, bool ONEBUF = false>
__global__ void __launch_bounds__(128 * NWG, MINB)
    fft_pass_kernel(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_out,
                    const KParams p) {
  using namespace dev;
  using C = Cfg<E, R1, R2, R3, MODE>;
  constexpr int S = C::S;
  constexpr int TM = C::TMAX;
  constexpr int T0 = C::T(0);
  constexpr int DH = T0 / 2 * C::NP(0);  // ONEBUF: stage-1 accumulator columns per half
  static_assert(!ONEBUF || (NWG == 1 && T0 % 2 == 0 && S >= 2 && DH + C::ACOLS <= 256 && C::DCOLS <= 256),
                "single-buffer geometry");
  constexpr uint32_t TCOLS = ONEBUF ? 256u : C::COLS;
  // Transposed-row passes write 16-byte runs whose merging in L2 is sensitive
  // to store timing: they keep the simple (lock-step) chunk loop, measured 1.6x
  // faster for them than the pipelined loop below (round 1).
  constexpr bool PIPE_OK = MODE != kModeRowT && MODE != kModeRowTB && S >= 2 && NWG == 1 && !ONEBUF;
  constexpr int NT = 128 * NWG;
  static_assert(C::T(0) % NWG == 0 && C::T(S - 1) % NWG == 0 && C::T(S > 1 ? 1 : 0) % NWG == 0, "NWG tiles");
  const bool PIPE = PIPE_OK && p.pipe;
  // Chunk schedule: a CTA's first chunk is blockIdx.x; later ones come from a
  // global ticket counter (thread 0, in load order), so CTAs on slower SMs
  // simply take fewer chunks (static striding left a 15 us tail on C2).  The
  // last CTA to retire resets the counter for the next launch.
  auto next_chunk = [&](int64_t cur) -> int64_t {
    if (!p.ctr || cur + gridDim.x < p.static_chunks) return cur + gridDim.x;
    const int64_t c = p.static_chunks + (int64_t)atomicAdd(p.ctr, 1ull);
    return c < p.chunks ? c : p.chunks;
  };

#ifndef TCFFT_NO_ALIGN_SLACK
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
#else
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
#endif
  uint8_t* s_in = smem;
  uint8_t* s_b = smem + p.smem_b;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.smem_bar);
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + 2);
  int64_t* s_q = reinterpret_cast<int64_t*>(bars + 4);  // chunk ids in load order (ring of 4)
  const int tid = threadIdx.x, warp = tid >> 5;
  const int wg = tid >> 7, ltid = tid & 127;  // warpgroup, TMEM lane / MMA row
  constexpr int TL0 = C::T(0) / NWG;
  const uint32_t s_in_u = smem_u32(s_in), s_b_u = smem_u32(s_b);

  // Thread 0 starts the first chunk's TMA load before anything else; the
  // other threads meanwhile stage the plan constants (B matrices, row
  // records).  Only thread 0 touches the transform's input/output (all data
  // movement is TMA), so only it waits on the preceding grid (PDL).
  // PDL trigger: at CTA start (pdl == 2), else as the CTA takes its last chunk
  if (p.pdl == 2 || (int64_t)blockIdx.x + gridDim.x >= p.chunks) griddep_launch_dependents();
  bool triggered = p.pdl == 2 || (int64_t)blockIdx.x + gridDim.x >= p.chunks;
  if (warp == 0) tmem_alloc<TCOLS>(s_tmem);
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    // tcgen05.commit (+ thread 0's arrive when pipelined; a second arrival in
    // the lock-step loop measured 1% slower on C2, round 1)
    mbar_init(&bars[1], PIPE ? 2 : 1);
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_in) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_out) : "memory");
#ifdef TCFFT_TRACE
    if (p.trace) p.trace[blockIdx.x * 8 + 0] = globaltimer_ns();
#endif
    griddep_wait();
#ifdef TCFFT_TRACE
    if (p.trace) p.trace[blockIdx.x * 8 + 1] = globaltimer_ns();
#endif
    if ((int64_t)blockIdx.x < p.chunks) issue_load<IoSet<MODE, TW4>::IN>(&tm_in, p.in, p.T, (int64_t)blockIdx.x, s_in, &bars[0]);
  }
  // constants: B matrices, once per CTA
  for (int i = tid; i < p.bbytes / 16; i += NT)
    reinterpret_cast<uint4*>(s_b)[i] = reinterpret_cast<const uint4*>(p.bblob)[i];

  // per-thread row records (host-built, see plan.cpp)
  auto rec = [&](int s, int t) -> const RowInfo& { return p.rows_tab[((size_t)s * p.tiles_max + t) * 128 + ltid]; };
  // stage-0 writers have c = 1; the final stage needs only its output address
  using RC = Rec<C, TW4>;
  constexpr bool RT = RC::IN_TMEM && NWG == 1 && !ONEBUF;
  constexpr int TMW = TM / NWG;
  // this thread's tiles: t = wg + NWG * tt
  int gb[TL0];
  int fk[TW4 ? C::T(S - 1) / NWG : 1];
  int waddr[S][TMW];
  float2 wc[S][TMW], ww[S][TMW];
#pragma unroll
  for (int tt = 0; tt < TL0; ++tt) gb[tt] = rec(0, wg + NWG * tt).gbase;
#pragma unroll
  for (int s = 0; s < S; ++s)
#pragma unroll
    for (int tt = 0; tt < TMW; ++tt) {
      if (tt < C::T(s) / NWG) {
        const RowInfo& r = rec(s, wg + NWG * tt);
        waddr[s][tt] = r.addr;
        if (s + 1 < S || TW4) ww[s][tt] = make_float2(r.wr, r.wi);
        if ((s >= 1 && s + 1 < S) || (TW4 && s + 1 == S)) wc[s][tt] = make_float2(r.cr, r.ci);
        if (TW4 && s + 1 == S) fk[tt] = r.mp;
      }
    }

  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *s_tmem;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t tD = tbase;
  const uint32_t tA = tbase + (uint32_t)(ONEBUF ? DH : C::DCOLS);
  const uint32_t tR = tbase + (uint32_t)RC::COL + lane_off;  // this lane's row records
  if constexpr (RT) {
    uint32_t w[RC::N];
#pragma unroll
    for (int t = 0; t < C::T(0); ++t) w[t] = (uint32_t)gb[t];
#pragma unroll
    for (int s = 0; s + 1 < S; ++s)
#pragma unroll
      for (int t = 0; t < C::T(s); ++t) {
        uint32_t* q = w + RC::OFF_W(s) + t * RC::WS(s);
        q[0] = (uint32_t)waddr[s][t];
        q[1] = __float_as_uint(ww[s][t].x);
        q[2] = __float_as_uint(ww[s][t].y);
        if (s >= 1) {
          q[3] = __float_as_uint(wc[s][t].x);
          q[4] = __float_as_uint(wc[s][t].y);
        }
      }
#pragma unroll
    for (int t = 0; t < C::T(S - 1); ++t) {
      uint32_t* q = w + RC::OFF_F + t * RC::FW;
      q[0] = (uint32_t)waddr[S - 1][t];
      if constexpr (TW4) {
        q[1] = (uint32_t)fk[t];
        q[2] = __float_as_uint(wc[S - 1][t].x);
        q[3] = __float_as_uint(wc[S - 1][t].y);
        q[4] = __float_as_uint(ww[S - 1][t].x);
        q[5] = __float_as_uint(ww[S - 1][t].y);
      }
    }
#pragma unroll
    for (int i = 0; i < RC::N; ++i) tmem_st1(tR + i, w + i);
    tmem_wait_st();
  }

  float2* s_tw4 = reinterpret_cast<float2*>(smem + p.smem_tw4);

  if (!PIPE) {
    // ------------------------------------------------------------ simple loop
    int64_t chunk = blockIdx.x;  // its load was issued in the prologue
    uint32_t ld_phase = 0, mma_phase = 0;
    // A operand / output staging: one buffer, or two alternating per chunk
    // (a_stride != 0: chunk i's writers only wait for chunk i-2's store)
    uint8_t* s_a = smem + p.smem_a;
    uint32_t s_a_u = smem_u32(s_a);
    // thread 0 takes chunk tickets one chunk ahead: the (dynamic) ticket's
    // atomic round trip overlaps a whole chunk instead of delaying the MMAs
    // (kept in shared memory, s_q[1]: a live register here costs spills)
    if (tid == 0 && p.ctr) s_q[1] = chunk < p.chunks ? next_chunk(chunk) : p.chunks;
#ifdef TCFFT_TRACE
    bool first = true;
#endif
    while (chunk < p.chunks) {
      mbar_wait(&bars[0], ld_phase);
      ld_phase ^= 1;
      // (single-buffer passes: the gather's TMEM stores reuse columns the
      // previous chunk's final epilogue read before the last barrier)
      if constexpr (ONEBUF) tc_fence_after();
#ifdef TCFFT_TRACE
      if (first && tid == 0 && p.trace) p.trace[blockIdx.x * 8 + 4] = globaltimer_ns();
#endif
      int g1[TL0];
      if constexpr (RT) {
        tmem_ld_words<C::T(0)>(tR, reinterpret_cast<uint32_t*>(g1));
        tmem_wait_ld();
      } else {
#pragma unroll
        for (int tt = 0; tt < TL0; ++tt) g1[tt] = gb[tt];
      }
#pragma unroll
      for (int tt = 0; tt < TL0; ++tt)
        gather_to_tmem<C>(s_in_u, g1[tt], p.gstride, (uint32_t)p.swz_in,
                          tA + lane_off + (wg + NWG * tt) * (C::KP(0) / 2));
      tmem_wait_st();
      tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        const int64_t nxt = p.ctr ? s_q[1] : chunk + gridDim.x;
        s_q[0] = nxt;  // read by all threads after this iteration's last barrier
        if (nxt < p.chunks) {
          // (single-buffer passes: issued after this chunk's store, below)
          if constexpr (!ONEBUF) issue_load<IoSet<MODE, TW4>::IN>(&tm_in, p.in, p.T, nxt, s_in, &bars[0]);  // staging buffer is free again
          if (p.ctr) s_q[1] = next_chunk(nxt);
        } else if (p.pdl == 1 && !triggered) {
          griddep_launch_dependents();  // this CTA's last chunk
        }
        if constexpr (ONEBUF) {
          issue_stage_mma<C, 0, 0, T0 / 2, true>(s_a_u, s_b_u, tD, tA);  // first half of stage 1
        } else {
          // the output store that last read this chunk's A buffer is done with it
          // (late_wait: stage 1 reads TMEM and the B matrices only, so its MMAs
          // are issued first and the wait overlaps them; the barrier below
          // holds the writers until thread 0 has passed it)
          if (!p.late_wait) {
            if (p.a_stride)
              bulk_wait_read1();
            else
              bulk_wait_read0();
          }
          issue_stage_mma<C, 0>(s_a_u, s_b_u, tD, tA);
        }
        mma_commit(&bars[1]);
        if (!ONEBUF && p.late_wait) {
          if (p.a_stride)
            bulk_wait_read1();
          else
            bulk_wait_read0();
        }
      }
      if constexpr (TW4) {
        // four-step twiddle, strip-base part: A[k] = W_Ntot^{base k}, r = W_Ntot^{base s}
        // (Ntot a power of two).  Computed by warps 1-3 while thread 0 issues the
        // stage-1 MMAs: the last chunk's final epilogue is done with s_tw4, this
        // chunk's reads it after the writer barrier(s).
        if (tid >= 32) {
          const int64_t base = ((chunk % p.in.spi) * (int64_t)p.in.C + p.tw4_col0) >> p.tw4_shift;
          for (int kk = tid - 32; kk <= p.tw4_nk; kk += NT - 32) {
            const int64_t e = (base * (kk < p.tw4_nk ? kk : p.tw4_s)) & (p.tw4_total - 1);
            float sn, cs;
            sincospif(-2.0f * (float)e / (float)p.tw4_total, &sn, &cs);
            s_tw4[kk] = make_float2(cs, sn);
          }
        }
        if constexpr (S == 1) __syncthreads();
      }
      mbar_wait(&bars[1], mma_phase);
      mma_phase ^= 1;
      if (!ONEBUF && p.late_wait) __syncthreads();
      tc_fence_after();
#ifdef TCFFT_TRACE
      if (first && tid == 0 && p.trace) p.trace[blockIdx.x * 8 + 5] = globaltimer_ns();
#endif
      auto writer = [&](auto sc) {
        constexpr int s = decltype(sc)::value;
        [[maybe_unused]] uint32_t rw[C::T(s) * RC::WS(s)];
        if constexpr (RT) {
          tmem_ld_words<C::T(s) * RC::WS(s)>(tR + RC::OFF_W(s), rw);
          tmem_wait_ld();
        }
#pragma unroll
        for (int tt = 0; tt < C::T(s) / NWG; ++tt) {
          int ad;
          float2 cc = make_float2(1.f, 0.f), wv;
          if constexpr (RT) {
            const uint32_t* q = rw + tt * RC::WS(s);
            ad = (int)q[0];
            wv = make_float2(__uint_as_float(q[1]), __uint_as_float(q[2]));
            if constexpr (s >= 1) cc = make_float2(__uint_as_float(q[3]), __uint_as_float(q[4]));
          } else {
            ad = waddr[s][tt];
            wv = ww[s][tt];
            if constexpr (s >= 1) cc = wc[s][tt];
          }
          writer_epilogue<C, s>(tD + lane_off + (wg + NWG * tt) * C::NP(s), s_a_u + ad, cc, wv);
        }
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
          tc_fence_after();
          issue_stage_mma<C, s + 1>(s_a_u, s_b_u, tD, tA);
          mma_commit(&bars[1]);
        }
        mbar_wait(&bars[1], mma_phase);
        mma_phase ^= 1;
        tc_fence_after();
      };
      if constexpr (ONEBUF) {
        // stage-1 writer in two halves over one accumulator region: half 0's
        // epilogue drains D, then the second half of stage 1 refills it
#pragma unroll
        for (int tt = 0; tt < T0 / 2; ++tt)
          writer_epilogue<C, 0>(tD + lane_off + tt * C::NP(0), s_a_u + waddr[0][tt], make_float2(1.f, 0.f),
                                ww[0][tt]);
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
          tc_fence_after();
          issue_stage_mma<C, 0, T0 / 2, T0, true>(s_a_u, s_b_u, tD, tA);
          mma_commit(&bars[1]);
        }
        mbar_wait(&bars[1], mma_phase);
        mma_phase ^= 1;
        tc_fence_after();
#pragma unroll
        for (int tt = T0 / 2; tt < T0; ++tt)
          writer_epilogue<C, 0>(tD + lane_off + (tt - T0 / 2) * C::NP(0), s_a_u + waddr[0][tt],
                                make_float2(1.f, 0.f), ww[0][tt]);
        fence_proxy_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
          tc_fence_after();
          issue_stage_mma<C, 1>(s_a_u, s_b_u, tD, tA);
          mma_commit(&bars[1]);
        }
        mbar_wait(&bars[1], mma_phase);
        mma_phase ^= 1;
        tc_fence_after();
      } else if constexpr (S >= 2) {
        writer(std::integral_constant<int, 0>{});
      }
      if constexpr (S >= 3) writer(std::integral_constant<int, 1>{});
      [[maybe_unused]] uint32_t rf[C::T(S - 1) * RC::FW];
      if constexpr (RT) {
        tmem_ld_words<C::T(S - 1) * RC::FW>(tR + RC::OFF_F, rf);
        tmem_wait_ld();
      }
#pragma unroll
      for (int tt = 0; tt < C::T(S - 1) / NWG; ++tt) {
        float2 c4 = make_float2(1.f, 0.f), w4 = make_float2(1.f, 0.f);
        int ad;
        if constexpr (RT)
          ad = (int)rf[tt * RC::FW];
        else
          ad = waddr[S - 1][tt];
        if constexpr (TW4) {
          int kk;
          float2 hc, hw;
          if constexpr (RT) {
            const uint32_t* q = rf + tt * RC::FW;
            kk = (int)q[1];
            hc = make_float2(__uint_as_float(q[2]), __uint_as_float(q[3]));
            hw = make_float2(__uint_as_float(q[4]), __uint_as_float(q[5]));
          } else {
            kk = fk[tt];
            hc = wc[S - 1][tt];
            hw = ww[S - 1][tt];
          }
          const float2 a = s_tw4[kk], r = s_tw4[p.tw4_nk];
          c4 = make_float2(a.x * hc.x - a.y * hc.y, a.x * hc.y + a.y * hc.x);
          w4 = make_float2(r.x * hw.x - r.y * hw.y, r.x * hw.y + r.y * hw.x);
        }
        final_epilogue<C, TW4>(tD + lane_off + (wg + NWG * tt) * C::NP(S - 1), s_a_u, ad, p.ostride,
                               (uint32_t)p.swz_out, c4, w4);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        issue_store<IoSet<MODE, TW4>::OUT, MODE == kModeStrip4>(&tm_out, p.out, p.T, chunk, s_a);
        if constexpr (ONEBUF) {
          // the buffer is free once the store has read it: load the next chunk
          if (s_q[0] < p.chunks) {
            bulk_wait_read0();
            issue_load<IoSet<MODE, TW4>::IN>(&tm_in, p.in, p.T, s_q[0], s_in, &bars[0]);
          }
        }
      }
#ifdef TCFFT_TRACE
      if (first && tid == 0 && p.trace) p.trace[blockIdx.x * 8 + 6] = globaltimer_ns();
      first = false;
#endif
      chunk = s_q[0];
      if (p.a_stride) {
        s_a = (s_a == smem + p.smem_a) ? s_a + p.a_stride : smem + p.smem_a;
        s_a_u = smem_u32(s_a);
      }
    }
  } else if constexpr (PIPE_OK) {
  // ---------------------------------------------------------------------
  // Software-pipelined chunk loop.  The MMA barrier (bars[1]) completes on two
  // arrivals: the tcgen05.commit of the stage's MMAs and a plain arrive by
  // thread 0 (issued after any wait thread 0 owes the other warps, e.g. the
  // previous output store releasing s_a), so thread 0 never delays MMA issue.
  // While the last stage's MMAs of chunk i run, all threads already gather
  // chunk i+1 into the (idle) stage-1 TMEM A region.
  uint32_t ld_phase = 0, mma_phase = 0;
  const int64_t chunk0 = blockIdx.x;
  auto rec_g1 = [&](int* g1) {
    if constexpr (RT) {
      tmem_ld_words<C::T(0)>(tR, reinterpret_cast<uint32_t*>(g1));
      tmem_wait_ld();
    } else {
#pragma unroll
      for (int t = 0; t < C::T(0); ++t) g1[t] = gb[t];
    }
  };
  auto tw4_table = [&](int64_t ch) {
    if constexpr (TW4) {
      // four-step twiddle, strip-base part: A[k] = W_Ntot^{base k}, r = W_Ntot^{base s}
      const int64_t base = ((ch % p.in.spi) * (int64_t)p.in.C + p.tw4_col0) >> p.tw4_shift;
      for (int kk = tid; kk <= p.tw4_nk; kk += 128) {
        const int64_t e = (base * (kk < p.tw4_nk ? kk : p.tw4_s)) % p.tw4_total;
        float sn, cs;
        sincospif(-2.0f * (float)e / (float)p.tw4_total, &sn, &cs);
        s_tw4[kk] = make_float2(cs, sn);
      }
    }
  };
  // stage-1 gather of `ch` (its TMA load must have been issued)
  auto gather = [&]() {
    mbar_wait(&bars[0], ld_phase);
    ld_phase ^= 1;
    int g1[C::T(0)];
    rec_g1(g1);
#pragma unroll
    for (int t = 0; t < C::T(0); ++t)
      gather_to_tmem<C>(s_in_u, g1[t], p.gstride, (uint32_t)p.swz_in, tA + lane_off + t * (C::KP(0) / 2));
    tmem_wait_st();
  };
  auto wait_mma = [&]() {
    mbar_wait(&bars[1], mma_phase);
    mma_phase ^= 1;
    tc_fence_after();
  };
  uint8_t* const s_a = smem + p.smem_a;
  const uint32_t s_a_u = smem_u32(s_a);

  if (chunk0 < p.chunks) {  // its load was issued in the prologue
    gather();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const int64_t c1 = next_chunk(chunk0);
      s_q[1] = c1;  // read after the first writer barrier of iteration 0
      if (c1 < p.chunks) issue_load<IoSet<MODE, TW4>::IN>(&tm_in, p.in, p.T, c1, s_in, &bars[0]);
      else if (p.pdl == 1 && !triggered) griddep_launch_dependents();
      issue_stage_mma<C, 0>(s_a_u, s_b_u, tD, tA);
      mma_commit(&bars[1]);
      mbar_arrive(&bars[1]);
    }
  }

  int64_t chunk = chunk0;
  for (int it = 0; chunk < p.chunks; ++it) {
    tw4_table(chunk);
    int64_t next = p.chunks;
    bool has_next = false;

    // ---------------- writer stages: wait MMA s, epilogue s, issue MMA s+1
    auto writer = [&](auto sc) {
      constexpr int s = decltype(sc)::value;
      wait_mma();
      [[maybe_unused]] uint32_t rw[C::T(s) * RC::WS(s)];
      if constexpr (RT) {
        tmem_ld_words<C::T(s) * RC::WS(s)>(tR + RC::OFF_W(s), rw);
        tmem_wait_ld();
      }
#pragma unroll
      for (int t = 0; t < C::T(s); ++t) {
        int ad;
        float2 cc = make_float2(1.f, 0.f), wv;
        if constexpr (RT) {
          const uint32_t* q = rw + t * RC::WS(s);
          ad = (int)q[0];
          wv = make_float2(__uint_as_float(q[1]), __uint_as_float(q[2]));
          if constexpr (s >= 1) cc = make_float2(__uint_as_float(q[3]), __uint_as_float(q[4]));
        } else {
          ad = waddr[s][t];
          wv = ww[s][t];
          if constexpr (s >= 1) cc = wc[s][t];
        }
        writer_epilogue<C, s>(tD + lane_off + t * C::NP(s), s_a_u + ad, cc, wv);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        issue_stage_mma<C, s + 1>(s_a_u, s_b_u, tD, tA);
        mma_commit(&bars[1]);
        mbar_arrive(&bars[1]);
      }
    };
    if constexpr (S >= 2) writer(std::integral_constant<int, 0>{});
    // the next chunk id (written by thread 0 before the barrier just passed)
    next = s_q[(it + 1) & 3];
    has_next = next < p.chunks;
    if constexpr (S >= 3) writer(std::integral_constant<int, 1>{});

    // ---------------- overlap: gather the next chunk while the last MMAs run
    // (single-stage plans: the last MMA reads the TMEM A region, wait first)
    if (S >= 2 && p.gather_ahead) {
      if (has_next) gather();
      wait_mma();
    } else {
      wait_mma();
      if (has_next) gather();
    }

    // ---------------- final epilogue -> output staging (reuses s_a)
    uint32_t rf[C::T(S - 1) * RC::FW];
    if constexpr (RT) {
      tmem_ld_words<C::T(S - 1) * RC::FW>(tR + RC::OFF_F, rf);
      tmem_wait_ld();
    }
#pragma unroll
    for (int t = 0; t < C::T(S - 1); ++t) {
      float2 c4 = make_float2(1.f, 0.f), w4 = make_float2(1.f, 0.f);
      int ad = RT ? (int)rf[t * RC::FW] : waddr[S - 1][t];
      if constexpr (TW4) {
        int kk;
        float2 hc, hw;
        if constexpr (RT) {
          const uint32_t* q = rf + t * RC::FW;
          kk = (int)q[1];
          hc = make_float2(__uint_as_float(q[2]), __uint_as_float(q[3]));
          hw = make_float2(__uint_as_float(q[4]), __uint_as_float(q[5]));
        } else {
          kk = fk[t];
          hc = wc[S - 1][t];
          hw = ww[S - 1][t];
        }
        const float2 a = s_tw4[kk], r = s_tw4[p.tw4_nk];
        c4 = make_float2(a.x * hc.x - a.y * hc.y, a.x * hc.y + a.y * hc.x);
        w4 = make_float2(r.x * hw.x - r.y * hw.y, r.x * hw.y + r.y * hw.x);
      }
      final_epilogue<C, TW4>(tD + lane_off + t * C::NP(S - 1), s_a_u, ad, p.ostride, (uint32_t)p.swz_out, c4, w4);
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      issue_store<IoSet<MODE, TW4>::OUT, MODE == kModeStrip4>(&tm_out, p.out, p.T, chunk, s_a);
      if (has_next) {
        // next chunk: its staging buffer is free (gathered above): prefetch the
        // one after, start its stage-1 MMAs, then release the epilogue warps
        // once the store just issued has finished reading s_a
        const int64_t n2 = next_chunk(next);
        s_q[(it + 2) & 3] = n2;
        if (n2 < p.chunks) issue_load<IoSet<MODE, TW4>::IN>(&tm_in, p.in, p.T, n2, s_in, &bars[0]);
        else if (p.pdl == 1 && !triggered) griddep_launch_dependents();
        issue_stage_mma<C, 0>(s_a_u, s_b_u, tD, tA);
        mma_commit(&bars[1]);
        bulk_wait_read0();
        mbar_arrive(&bars[1]);
      }
    }
    chunk = next;
  }
  }  // PIPE
  if (tid == 0) {
#ifdef TCFFT_TRACE
    if (p.trace) p.trace[blockIdx.x * 8 + 7] = globaltimer_ns();
#endif
    bulk_wait0();
    if (p.ctr) {
      __threadfence();
      if (atomicAdd(p.ctr + 1, 1ull) == gridDim.x - 1) {  // last CTA out: reset for the next launch
        p.ctr[0] = 0;
        p.ctr[1] = 0;
        __threadfence();
      }
    }
  }
#ifdef TCFFT_TRACE
  if (p.trace && tid == 0) {
    p.trace[blockIdx.x * 8 + 2] = globaltimer_ns();
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    p.trace[blockIdx.x * 8 + 3] = sm;
  }
#endif
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<TCOLS>(tbase);
}

}  // namespace tcfft
