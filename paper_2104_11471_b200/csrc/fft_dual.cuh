// fft_dual.cuh - dual-context pass kernel for 16384-element chunks.
//
// A 16384-element chunk (a 2048 x 8 / 4096 x 4 / 1024 x 16 column strip, 8
// rows of 2048, one 16384-point row) needs 64 KB of staging and 64 KB of
// A-operand / output staging, so the plain kernel fits ONE CTA per SM, and
// that CTA's load -> MMA -> epilogue -> barrier chain leaves the SM idle
// most of the time (0.56 - 0.68 of the HBM roofline, round 1/2).  Here one
// CTA of two warpgroups runs two chunk CONTEXTS concurrently:
//
//   * shared-memory: one staging buffer Z shared by the contexts (TMA load ->
//     stage-1 gather), one A / output buffer X_w per context, the DFT
//     matrices once (radix >= 32 planar stages keep only Fr and Fi: the
//     -Fi block is the instruction descriptor's negate-B bit), twiddle tables
//     per context: 64 + 2 x 65 + <= 20 KB;
//   * tensor memory: 256 columns per context (stage 1 runs in two halves of
//     tiles over one accumulator region, later stages reuse the dead stage-1
//     A operand's columns);
//   * chunks of the CTA alternate between the contexts; the context that has
//     just gathered chunk i from Z loads chunk i + 1 into Z for the other
//     context (zfull[i % 2] signals it), so the next load overlaps both
//     contexts' MMAs and epilogues, and one context's MMA latency overlaps the
//     other context's epilogue work.
//
// Each context synchronises with its own named barrier (bar.sync 1 + w, 128)
// and its own MMA mbarrier; the contexts only share Z, the B matrices and the
// chunk-id slots.  HBM is touched once per element per pass, as in
// fft_kernel.cuh.
#pragma once
#include "fft_kernel.cuh"

namespace tcfft {
namespace dev {

// DFT matrices of the dual kernel (plan.cpp build_bblob mirrors this layout).
template <class C>
struct DualB {
  __host__ __device__ static constexpr bool PLANAR(int s) { return s >= 1 || C::PLANAR0; }
  // halved: Fr and Fi (R x R each, K-major canonical, N = R)
  __host__ __device__ static constexpr bool HB(int s) { return PLANAR(s) && C::R(s) >= 32; }
  __host__ __device__ static constexpr int SZ(int s) { return HB(s) ? 4 * C::R(s) * C::R(s) : C::KP(s) * C::NP(s) * 2; }
  __host__ __device__ static constexpr bool SHARE(int s) {
    return s >= 1 && PLANAR(s) && PLANAR(s - 1) && C::R(s) == C::R(s - 1);
  }
  __host__ __device__ static constexpr int END(int s) { return s < 0 ? 0 : (SHARE(s) ? END(s - 1) : OFF(s) + SZ(s)); }
  __host__ __device__ static constexpr int OFF(int s) { return s == 0 ? 0 : (SHARE(s) ? OFF(s - 1) : END(s - 1)); }
};

DEVI void ctx_sync(int w) { asm volatile("bar.sync %0, 128;" ::"r"(1 + w) : "memory"); }

// MMAs of stage s for tiles [TB, TE) (accumulators at (t - TB) * NP when
// DSHIFT), one elected thread.
template <class C, int s, int TB, int TE, bool DSHIFT>
DEVI void dual_stage_mma(uint32_t s_a, uint32_t s_b, uint32_t tD, uint32_t tA) {
  using B = DualB<C>;
  constexpr int KP = C::KP(s), NP = C::NP(s), R = C::R(s);
  constexpr uint32_t amn = s == 0 ? 0u : 1u;  // stage 1: A from TMEM (K-major); later: SMEM MN-major
#pragma unroll
  for (int t = TB; t < TE; ++t) {
    const uint32_t dcol = tD + (DSHIFT ? t - TB : t) * NP;
    auto adesc = [&](int q) -> uint64_t { return make_sdesc(s_a + t * C::TILEB(s) + q * 256, 128, C::SBO(s)); };
    if constexpr (!B::HB(s)) {
      constexpr uint32_t idesc = make_idesc_f16(128, NP, amn, 0);
#pragma unroll
      for (int q = 0; q < KP / 16; ++q) {
        const uint64_t bd = make_sdesc(s_b + B::OFF(s) + q * 32 * NP, 128, 256);
        if constexpr (s == 0)
          mma_ts(dcol, tA + t * (KP / 2) + q * 8, bd, idesc, q > 0);
        else
          mma_ss(dcol, adesc(q), bd, idesc, q > 0);
      }
    } else {
      // D_re = xr Fr + xi (-Fi), D_im = xr Fi + xi Fr over planar K (re | im)
      constexpr uint32_t idesc = make_idesc_f16(128, R, amn, 0);
      constexpr uint32_t NEGB = 1u << 14;
#pragma unroll
      for (int cout = 0; cout < 2; ++cout)
#pragma unroll
        for (int q = 0; q < KP / 16; ++q) {
          const int cin = q / (R / 16), kq = q % (R / 16);
          const bool fi = cin != cout;
          const uint64_t bd = make_sdesc(s_b + B::OFF(s) + (fi ? 2 * R * R : 0) + kq * 32 * R, 128, 256);
          const uint32_t id = idesc | ((cin == 1 && cout == 0) ? NEGB : 0u);
          if constexpr (s == 0)
            mma_ts(dcol + cout * R, tA + t * (KP / 2) + q * 8, bd, id, q > 0);
          else
            mma_ss(dcol + cout * R, adesc(q), bd, id, q > 0);
        }
    }
  }
}

}  // namespace dev

template <int E, int R1, int R2, int R3, int MODE, bool TW4>
__global__ void __launch_bounds__(256, 1)
    fft_dual_kernel(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_out,
                    const KParams p) {
  using namespace dev;
  using C = Cfg<E, R1, R2, R3, MODE>;
  using B = DualB<C>;
  constexpr int S = C::S;
  constexpr int TM = C::TMAX;
  constexpr int T0 = C::T(0);
  constexpr int DH = T0 / 2 * C::NP(0);
  static_assert(S >= 2 && T0 % 2 == 0 && DH + C::ACOLS <= 256 && C::DCOLS <= 256, "dual geometry");

  auto next_chunk = [&](int64_t cur) -> int64_t {
    if (!p.ctr || cur + gridDim.x < p.static_chunks) return cur + gridDim.x;
    const int64_t c = p.static_chunks + (int64_t)atomicAdd(p.ctr, 1ull);
    return c < p.chunks ? c : p.chunks;
  };

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5;
  const int w = tid >> 7, ltid = tid & 127;  // context, TMEM lane / MMA row
  const bool lead = ltid == 0;
  uint8_t* s_z = smem;
  uint8_t* s_x = smem + p.smem_a + w * p.a_stride;
  uint8_t* s_b = smem + p.smem_b;
  const int tw4_bytes = ((p.tw4_nk * 8 + 16 + 127) & ~127);
  float2* s_tw4 = reinterpret_cast<float2*>(smem + p.smem_tw4 + w * tw4_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + p.smem_bar);  // zfull[2], mma[2]
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + 4);
  volatile int64_t* s_q = reinterpret_cast<int64_t*>(bars + 6);  // chunk id per context
  const uint32_t s_z_u = smem_u32(s_z), s_x_u = smem_u32(s_x), s_b_u = smem_u32(s_b);

  bool triggered = p.pdl == 2 || (int64_t)blockIdx.x + gridDim.x >= p.chunks;
  if (triggered) griddep_launch_dependents();
  if (warp == 0) tmem_alloc<512>(s_tmem);
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_in) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tm_out) : "memory");
    griddep_wait();
    s_q[0] = blockIdx.x;  // grid <= chunks
    issue_load(&tm_in, p.in, p.T, (int64_t)blockIdx.x, s_z, &bars[0]);
  }
  for (int i = tid; i < p.bbytes / 16; i += 256)
    reinterpret_cast<uint4*>(s_b)[i] = reinterpret_cast<const uint4*>(p.bblob)[i];

  // per-thread row records (host-built, plan.cpp): every tile of every stage
  auto rec = [&](int s, int t) -> const RowInfo& { return p.rows_tab[((size_t)s * p.tiles_max + t) * 128 + ltid]; };
  int gb[T0];
  int fk[TW4 ? C::T(S - 1) : 1];
  int waddr[S][TM];
  float2 wc[S][TM], ww[S][TM];
#pragma unroll
  for (int t = 0; t < T0; ++t) gb[t] = rec(0, t).gbase;
#pragma unroll
  for (int s = 0; s < S; ++s)
#pragma unroll
    for (int t = 0; t < TM; ++t) {
      if (t < C::T(s)) {
        const RowInfo& r = rec(s, t);
        waddr[s][t] = r.addr;
        if (s + 1 < S || TW4) ww[s][t] = make_float2(r.wr, r.wi);
        if ((s >= 1 && s + 1 < S) || (TW4 && s + 1 == S)) wc[s][t] = make_float2(r.cr, r.ci);
        if (TW4 && s + 1 == S) fk[t] = r.mp;
      }
    }

  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t tD = *s_tmem + (uint32_t)(w * 256);
  const uint32_t tA = tD + (uint32_t)DH;
  uint64_t* zfull = &bars[w];
  uint64_t* mbar = &bars[2 + w];
  uint32_t ph_z = 0, ph_m = 0;

  auto wait_mma = [&]() {
    mbar_wait(mbar, ph_m);
    ph_m ^= 1;
    tc_fence_after();
  };
  // end of a stage's epilogue: the next MMAs may read what it wrote
  auto stage_done = [&](bool smem_written) {
    if (smem_written) fence_proxy_async_smem();
    tc_fence_before();
    ctx_sync(w);
  };

  while (true) {
    mbar_wait(zfull, ph_z);
    ph_z ^= 1;
    const int64_t chunk = s_q[w];
    if (chunk >= p.chunks) {
      // no more chunks: wake the other context (it may be waiting for a load
      // that will never come) with the same sentinel, then leave
      if (lead) {
        s_q[1 - w] = p.chunks;
        mbar_arrive(&bars[1 - w]);
      }
      break;
    }
    tc_fence_after();
    // ---- stage-1 gather: Z -> this context's TMEM A operand
#pragma unroll
    for (int t = 0; t < T0; ++t)
      gather_to_tmem<C>(s_z_u, gb[t], p.gstride, (uint32_t)p.swz_in, tA + lane_off + t * (C::KP(0) / 2));
    tmem_wait_st();
    tc_fence_before();
    ctx_sync(w);
    if (lead) {
      tc_fence_after();
      // Z is free: load the CTA's next chunk for the other context
      const int64_t nxt = next_chunk(chunk);
      if (nxt < p.chunks) {
        s_q[1 - w] = nxt;
        issue_load(&tm_in, p.in, p.T, nxt, s_z, &bars[1 - w]);
      } else {
        s_q[1 - w] = p.chunks;
        mbar_arrive(&bars[1 - w]);
        if (p.pdl == 1 && !triggered) griddep_launch_dependents();
      }
      bulk_wait_read0();  // this context's previous store has read X
      dual_stage_mma<C, 0, 0, T0 / 2, true>(s_x_u, s_b_u, tD, tA);
      mma_commit(mbar);
    }
    if constexpr (TW4) {
      // four-step twiddle, strip-base part (fft_kernel.cuh), per context
      if (ltid >= 32) {
        const int64_t base = ((chunk % p.in.spi) * (int64_t)p.in.C) >> p.tw4_shift;
        for (int kk = ltid - 32; kk <= p.tw4_nk; kk += 96) {
          const int64_t e = (base * (kk < p.tw4_nk ? kk : p.tw4_s)) & (p.tw4_total - 1);
          float sn, cs;
          sincospif(-2.0f * (float)e / (float)p.tw4_total, &sn, &cs);
          s_tw4[kk] = make_float2(cs, sn);
        }
      }
    }
    // ---- stage 1 in two halves over one accumulator region
    wait_mma();
#pragma unroll
    for (int t = 0; t < T0 / 2; ++t)
      writer_epilogue<C, 0>(tD + lane_off + t * C::NP(0), s_x_u + waddr[0][t], make_float2(1.f, 0.f), ww[0][t]);
    stage_done(false);
    if (lead) {
      tc_fence_after();
      dual_stage_mma<C, 0, T0 / 2, T0, true>(s_x_u, s_b_u, tD, tA);
      mma_commit(mbar);
    }
    wait_mma();
#pragma unroll
    for (int t = T0 / 2; t < T0; ++t)
      writer_epilogue<C, 0>(tD + lane_off + (t - T0 / 2) * C::NP(0), s_x_u + waddr[0][t], make_float2(1.f, 0.f),
                            ww[0][t]);
    stage_done(true);
    if (lead) {
      tc_fence_after();
      dual_stage_mma<C, 1, 0, C::T(1), false>(s_x_u, s_b_u, tD, tA);
      mma_commit(mbar);
    }
    wait_mma();
    if constexpr (S >= 3) {
#pragma unroll
      for (int t = 0; t < C::T(1); ++t)
        writer_epilogue<C, 1>(tD + lane_off + t * C::NP(1), s_x_u + waddr[1][t], wc[1][t], ww[1][t]);
      stage_done(true);
      if (lead) {
        tc_fence_after();
        dual_stage_mma<C, 2, 0, C::T(2), false>(s_x_u, s_b_u, tD, tA);
        mma_commit(mbar);
      }
      wait_mma();
    }
    // ---- final epilogue -> X (output staging), then the TMA store
#pragma unroll
    for (int t = 0; t < C::T(S - 1); ++t) {
      float2 c4 = make_float2(1.f, 0.f), w4 = make_float2(1.f, 0.f);
      if constexpr (TW4) {
        const float2 a = s_tw4[fk[t]], r = s_tw4[p.tw4_nk];
        const float2 hc = wc[S - 1][t], hw = ww[S - 1][t];
        c4 = make_float2(a.x * hc.x - a.y * hc.y, a.x * hc.y + a.y * hc.x);
        w4 = make_float2(r.x * hw.x - r.y * hw.y, r.x * hw.y + r.y * hw.x);
      }
      final_epilogue<C, TW4>(tD + lane_off + t * C::NP(S - 1), s_x_u, waddr[S - 1][t], p.ostride,
                             (uint32_t)p.swz_out, c4, w4);
    }
    stage_done(true);
    if (lead) issue_store<MODE == kModeStrip4>(&tm_out, p.out, p.T, chunk, s_x);
  }
  if (lead) bulk_wait0();
  __syncthreads();
  if (tid == 0 && p.ctr) {
    __threadfence();
    if (atomicAdd(p.ctr + 1, 1ull) == gridDim.x - 1) {  // last CTA out: reset for the next launch
      p.ctr[0] = 0;
      p.ctr[1] = 0;
      __threadfence();
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(*s_tmem);
}

}  // namespace tcfft
