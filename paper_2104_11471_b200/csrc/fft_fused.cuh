// fft_fused.cuh - one persistent launch for a two-pass transform (2D rows then
// columns; four-step column then row pass), with the batch walked in
// L2-sized groups so that the intermediate data written by pass A is consumed
// by pass B while it is still resident in L2: HBM sees (close to) one read
// and one write per element instead of two of each.
//
// Work items are chunks of either pass, ordered group by group with pass B of
// group g scheduled after pass A of group g + LAG:
//     A(0) .. A(LAG-1), [A(g+LAG), B(g)] for g = 0.., B(G-LAG) .. B(G-1)
// A pass-B chunk of object o (image / transform) depends on every pass-A chunk
// of o: pass-A chunks publish completion with a release add on a per-object
// counter once their TMA store has fully completed; a pass-B chunk's loader
// acquires the counter before issuing its TMA load.  Every CTA walks its items
// in increasing order and the grid is co-resident, so the dependency graph is
// acyclic and waits are short (the LAG keeps them off the critical path).
#pragma once
#include "fft_kernel.cuh"

namespace tcfft {

struct FusedParams {
  KParams a, b;
  unsigned long long* next_item;  // dynamic scheduler (zeroed before launch); null -> static round-robin
  int64_t items;
  int64_t groups;
  int32_t lag;
  int32_t objs_per_group;
  int32_t a_per_obj, b_per_obj;  // chunks of each pass per object
  int64_t objs;
  int32_t* counters;             // per object, monotonically increasing across executions
  int32_t epoch_base;            // counters reach epoch_base + a_per_obj in this execution
  int32_t smem_a_b;              // pass B's B-matrix blob offset (pass A: a.smem_b)
};

namespace dev {

// One pass's per-thread row records and chunk-stage code.  With COL >= 0 the
// records live in TMEM columns [COL, COL + Rec::N) of the thread's lane
// (loaded with tcgen05.ld where needed) instead of registers.
template <int E_, int R1_, int R2_, int R3_, int MODE_, bool TW4_, int COL_ = -1>
struct PassT {
  using C = Cfg<E_, R1_, R2_, R3_, MODE_>;
  using RC = Rec<C, TW4_>;
  static constexpr bool TW4 = TW4_;
  static constexpr bool RT = COL_ >= 0;
  static constexpr int S = C::S, TM = C::TMAX;
  int gb[RT ? 1 : C::T(0)];
  int fk[(TW4 && !RT) ? C::T(S - 1) : 1];
  int waddr[RT ? 1 : S][RT ? 1 : TM];
  float2 wc[RT ? 1 : S][RT ? 1 : TM], ww[RT ? 1 : S][RT ? 1 : TM];
  uint32_t tR = 0;

  // Fetch this thread's records from global; RT: park them in TMEM.
  DEVI void load(const KParams& p, int tid, uint32_t tbase_lane) {
    auto rec = [&](int s, int t) -> const RowInfo& { return p.rows_tab[((size_t)s * p.tiles_max + t) * 128 + tid]; };
    if constexpr (RT) {
      tR = tbase_lane + (uint32_t)COL_;
      uint32_t w[RC::N];
#pragma unroll
      for (int t = 0; t < C::T(0); ++t) w[t] = (uint32_t)rec(0, t).gbase;
#pragma unroll
      for (int s = 0; s + 1 < S; ++s)
#pragma unroll
        for (int t = 0; t < C::T(s); ++t) {
          const RowInfo& r = rec(s, t);
          uint32_t* q = w + RC::OFF_W(s) + t * RC::WS(s);
          q[0] = (uint32_t)r.addr;
          q[1] = __float_as_uint(r.wr);
          q[2] = __float_as_uint(r.wi);
          if (s >= 1) {
            q[3] = __float_as_uint(r.cr);
            q[4] = __float_as_uint(r.ci);
          }
        }
#pragma unroll
      for (int t = 0; t < C::T(S - 1); ++t) {
        const RowInfo& r = rec(S - 1, t);
        uint32_t* q = w + RC::OFF_F + t * RC::FW;
        q[0] = (uint32_t)r.addr;
        if constexpr (TW4) {
          q[1] = (uint32_t)r.mp;
          q[2] = __float_as_uint(r.cr);
          q[3] = __float_as_uint(r.ci);
          q[4] = __float_as_uint(r.wr);
          q[5] = __float_as_uint(r.wi);
        }
      }
#pragma unroll
      for (int i = 0; i < RC::N; ++i) tmem_st1(tR + i, w + i);
      tmem_wait_st();
    } else {
#pragma unroll
      for (int t = 0; t < C::T(0); ++t) gb[t] = rec(0, t).gbase;
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
    }
  }

  DEVI void gather(const KParams& p, uint32_t s_in_u, uint32_t tA_lane) const {
    int g[C::T(0)];
    if constexpr (RT) {
      tmem_ld_words<C::T(0)>(tR, reinterpret_cast<uint32_t*>(g));
      tmem_wait_ld();
    } else {
#pragma unroll
      for (int t = 0; t < C::T(0); ++t) g[t] = gb[t];
    }
#pragma unroll
    for (int t = 0; t < C::T(0); ++t)
      gather_to_tmem<C>(s_in_u, g[t], p.gstride, (uint32_t)p.swz_in, tA_lane + t * (C::KP(0) / 2));
    tmem_wait_st();
  }

  template <int s>
  DEVI void writer(uint32_t tD_lane, uint32_t s_a_u) const {
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
      writer_epilogue<C, s>(tD_lane + t * C::NP(s), s_a_u + ad, cc, wv);
    }
  }

  DEVI void final(const KParams& p, uint32_t tD_lane, uint32_t s_a_u, const float2* s_tw4) const {
    [[maybe_unused]] uint32_t rf[C::T(S - 1) * RC::FW];
    if constexpr (RT) {
      tmem_ld_words<C::T(S - 1) * RC::FW>(tR + RC::OFF_F, rf);
      tmem_wait_ld();
    }
#pragma unroll
    for (int t = 0; t < C::T(S - 1); ++t) {
      float2 c4 = make_float2(1.f, 0.f), w4 = make_float2(1.f, 0.f);
      int ad;
      if constexpr (RT)
        ad = (int)rf[t * RC::FW];
      else
        ad = waddr[S - 1][t];
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
      final_epilogue<C, TW4>(tD_lane + t * C::NP(S - 1), s_a_u, ad, p.ostride, (uint32_t)p.swz_out, c4, w4);
    }
  }
};

// TMEM column where pass B's records start when both passes park theirs in
// TMEM (A's start at the larger of the two working regions).
template <class CA, class CB, bool TWA, bool TWB>
struct FusedRec {
  static constexpr int WORK = (CA::DCOLS + CA::ACOLS) > (CB::DCOLS + CB::ACOLS) ? (CA::DCOLS + CA::ACOLS)
                                                                                 : (CB::DCOLS + CB::ACOLS);
  static constexpr uint32_t COLS = CA::COLS > CB::COLS ? CA::COLS : CB::COLS;
  static constexpr int NA = Rec<CA, TWA>::N, NB = Rec<CB, TWB>::N;
  static constexpr bool FIT = WORK + NA + NB <= (int)COLS;
  static constexpr int COL_A = FIT ? WORK : -1;
  static constexpr int COL_B = FIT ? WORK + NA : -1;
};

DEVI void signal_obj(int32_t* ctr) {
  asm volatile("fence.proxy.async.global;" ::: "memory");
  asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(ctr) : "memory");
}
DEVI void wait_obj(const int32_t* ctr, int32_t target) {
  int32_t v;
  while (true) {
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    if (v - target >= 0) break;
    __nanosleep(64);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// item -> (is pass B, pass-local chunk index)
DEVI void decode_item(const FusedParams& f, int64_t item, bool& isb, int64_t& chunk) {
  const int64_t na = (int64_t)f.objs_per_group * f.a_per_obj;  // pass-A chunks per group
  const int64_t nb = (int64_t)f.objs_per_group * f.b_per_obj;
  const int64_t head = f.lag * na;  // first LAG groups: pass A only
  if (item < head) {
    isb = false;
    chunk = item;
    return;
  }
  int64_t r = item - head;
  const int64_t mid_groups = f.groups - f.lag;  // slots holding A(g+LAG) then B(g)
  if (r < mid_groups * (na + nb)) {
    const int64_t g = r / (na + nb), o = r % (na + nb);
    if (o < na) {
      isb = false;
      chunk = (g + f.lag) * na + o;
    } else {
      isb = true;
      chunk = g * nb + (o - na);
    }
    return;
  }
  r -= mid_groups * (na + nb);
  isb = true;
  chunk = (mid_groups)*nb + r;
}

}  // namespace dev

// Fused two-pass persistent kernel, warp-specialised: warps 0-3 (128 threads,
// one per TMEM lane) run the FFT stages; warp 4 is the producer that issues
// the TMA loads and stores, resolves pass-B dependencies and publishes pass-A
// completions, so none of that latency sits on the compute warps' path.
//   full   : load landed (tx bytes)             producer -> compute
//   empty  : staging buffer gathered            compute  -> producer
//   ofull  : output staging written             compute  -> producer
//   oempty : output staging read by the store   producer -> compute
//   mma    : tcgen05.commit                      tensor   -> compute
template <class PA, class PB, int MINB>
__global__ void __launch_bounds__(160, MINB)
    fft_fused_kernel(const __grid_constant__ CUtensorMap ta_in, const __grid_constant__ CUtensorMap ta_out,
                     const __grid_constant__ CUtensorMap tb_in, const __grid_constant__ CUtensorMap tb_out,
                     const FusedParams f) {
  using namespace dev;
  using CA = typename PA::C;
  using CB = typename PB::C;
  constexpr uint32_t COLS = CA::COLS > CB::COLS ? CA::COLS : CB::COLS;
  const KParams& pa = f.a;
  const KParams& pb = f.b;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* s_in = smem;
  uint8_t* s_a = smem + pa.smem_a;  // both passes use the same A / staging offset
  uint8_t* s_ba = smem + pa.smem_b;
  uint8_t* s_bb = smem + f.smem_a_b;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + pa.smem_bar);  // 5 mbarriers + TMEM address
  uint64_t* b_full = bars + 0;
  uint64_t* b_mma = bars + 1;
  uint64_t* b_empty = bars + 2;
  uint64_t* b_ofull = bars + 3;
  uint64_t* b_oempty = bars + 4;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + 5);
  volatile int64_t* s_item = reinterpret_cast<volatile int64_t*>(bars + 6);  // ring of 2 item indices
  float2* s_tw4 = reinterpret_cast<float2*>(smem + pa.smem_tw4);
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t s_in_u = smem_u32(s_in), s_a_u = smem_u32(s_a), s_ba_u = smem_u32(s_ba), s_bb_u = smem_u32(s_bb);

  for (int i = tid; i < pa.bbytes / 16; i += 160)
    reinterpret_cast<uint4*>(s_ba)[i] = reinterpret_cast<const uint4*>(pa.bblob)[i];
  for (int i = tid; i < pb.bbytes / 16; i += 160)
    reinterpret_cast<uint4*>(s_bb)[i] = reinterpret_cast<const uint4*>(pb.bblob)[i];
  if (warp == 0) tmem_alloc<COLS>(s_tmem);
  if (tid == 128) {  // producer lane: the first two items
    int64_t i0 = f.next_item ? (int64_t)atomicAdd(f.next_item, 1ull) : (int64_t)blockIdx.x;
    if (i0 > f.items) i0 = f.items;
    int64_t i1 = i0 >= f.items ? f.items
                               : (f.next_item ? (int64_t)atomicAdd(f.next_item, 1ull) : i0 + (int64_t)gridDim.x);
    s_item[0] = i0;
    s_item[1] = i1 > f.items ? f.items : i1;
  }
  if (tid == 0) {
    mbar_init(b_full, 1);
    mbar_init(b_mma, 1);
    mbar_init(b_empty, 1);
    mbar_init(b_ofull, 1);
    mbar_init(b_oempty, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *s_tmem;

  if (warp == 4) {
    // ============================ producer warp ============================
    if ((tid & 31) == 0) {
      constexpr int DEPTH = 2;
      int64_t pend[DEPTH] = {-1, -1};
      int npend = 0;
      auto flush = [&]() {
        if (npend) {
          bulk_wait0();
          for (int i = 0; i < npend; ++i)
            if (pend[i] >= 0) signal_obj(f.counters + pend[i]);
          npend = 0;
        }
      };
      auto after_store = [&](int64_t obj) {
        if (npend == DEPTH) {
          asm volatile("cp.async.bulk.wait_group 2;" ::: "memory");
          if (pend[0] >= 0) signal_obj(f.counters + pend[0]);
          pend[0] = pend[1];
          npend = 1;
        }
        pend[npend++] = obj;
      };
      auto load = [&](int64_t item, bool block) -> bool {
        bool isb;
        int64_t ch;
        decode_item(f, item, isb, ch);
        if (isb) {
          const int32_t* ctr = f.counters + ch / f.b_per_obj;
          const int32_t target = f.epoch_base + f.a_per_obj;
          int32_t v;
          asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
          if (v - target < 0) {
            if (!block) return false;
            flush();
            wait_obj(ctr, target);
          }
          asm volatile("fence.proxy.async.global;" ::: "memory");
          issue_load(&tb_in, pb.in, pb.T, ch, s_in, b_full);
        } else {
          issue_load(&ta_in, pa.in, pa.T, ch, s_in, b_full);
        }
        return true;
      };
      uint32_t ph_empty = 0, ph_ofull = 0;
      auto grab = [&](int64_t cur) -> int64_t {
        if (cur >= f.items) return f.items;
        if (f.next_item) return (int64_t)atomicAdd(f.next_item, 1ull);
        return cur + gridDim.x;
      };
      // item j's index sits in s_item[j & 1]; the compute warps read item
      // j+1's at the end of item j, after thread 0 observed oempty(j-1), which
      // this warp arrives only after writing it.
      int64_t cur = s_item[0], nxt = s_item[1];
      int j = 0;
      if (cur < f.items) load(cur, true);
      while (cur < f.items) {
        bool isb;
        int64_t ch;
        decode_item(f, cur, isb, ch);
        mbar_wait(b_empty, ph_empty);  // staging gathered: prefetch the next item
        ph_empty ^= 1;
        const bool loaded = nxt < f.items ? load(nxt, false) : true;
        const int64_t nxt2 = grab(nxt);
        s_item[(j + 2) & 1] = nxt2;
        mbar_wait(b_ofull, ph_ofull);  // output staging written
        ph_ofull ^= 1;
        issue_store(isb ? &tb_out : &ta_out, isb ? pb.out : pa.out, isb ? pb.T : pa.T, ch, s_a);
        bulk_wait_read0();
        mbar_arrive(b_oempty);  // compute warps may overwrite s_a
        after_store(isb ? -1 : ch / f.a_per_obj);
        if (!loaded) load(nxt, true);
        cur = nxt;
        nxt = nxt2;
        ++j;
      }
      flush();
      bulk_wait0();
    }
  } else {
    // ============================ compute warps ============================
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    const uint32_t tD = tbase;
    const uint32_t tAA = tbase + (uint32_t)CA::DCOLS, tAB = tbase + (uint32_t)CB::DCOLS;
    PA A;
    PB B;
    A.load(pa, tid, tbase + lane_off);
    B.load(pb, tid, tbase + lane_off);
    uint32_t ph_full = 0, ph_mma = 0, ph_oempty = 0;
    bool first_item = true;
    auto csync = []() { asm volatile("bar.sync 1, 128;" ::: "memory"); };  // compute warps only
    auto wait_mma = [&]() {
      mbar_wait(b_mma, ph_mma);
      ph_mma ^= 1;
      tc_fence_after();
    };
    auto run = [&](auto& P, const KParams& p, uint32_t tA, uint32_t s_b_u, int64_t ch) {
      using PT = std::remove_reference_t<decltype(P)>;
      using C = typename PT::C;
      constexpr int S = C::S;
      if constexpr (PT::TW4) {
        const int64_t base = ((ch % p.in.spi) * (int64_t)p.in.C) >> p.tw4_shift;
        for (int kk = tid; kk <= p.tw4_nk; kk += 128) {
          const int64_t e = (base * (kk < p.tw4_nk ? kk : p.tw4_s)) % p.tw4_total;
          float sn, cs;
          sincospif(-2.0f * (float)e / (float)p.tw4_total, &sn, &cs);
          s_tw4[kk] = make_float2(cs, sn);
        }
      }
      mbar_wait(b_full, ph_full);
      ph_full ^= 1;
      P.gather(p, s_in_u, tA + lane_off);
      tc_fence_before();
      csync();
      if (tid == 0) {
        mbar_arrive(b_empty);  // staging buffer free for the next load
        tc_fence_after();
        if (!first_item) {  // the previous store has finished reading s_a
          mbar_wait(b_oempty, ph_oempty);
        }
        issue_stage_mma<C, 0>(s_a_u, s_b_u, tD, tA);
        mma_commit(b_mma);
      }
      if (!first_item) ph_oempty ^= 1;
      first_item = false;
      auto writer = [&](auto sc) {
        constexpr int s = decltype(sc)::value;
        wait_mma();
        P.template writer<s>(tD + lane_off, s_a_u);
        fence_proxy_async_smem();
        tc_fence_before();
        csync();
        if (tid == 0) {
          tc_fence_after();
          issue_stage_mma<C, s + 1>(s_a_u, s_b_u, tD, tA);
          mma_commit(b_mma);
        }
      };
      if constexpr (S >= 2) writer(std::integral_constant<int, 0>{});
      if constexpr (S >= 3) writer(std::integral_constant<int, 1>{});
      wait_mma();
      P.final(p, tD + lane_off, s_a_u, s_tw4);
      fence_proxy_async_smem();
      tc_fence_before();
      csync();
      if (tid == 0) mbar_arrive(b_ofull);
    };
    // the producer writes item i+1's index into s_item before releasing item
    // i's ofull wait, i.e. before this loop reads it (csync orders the read)
    int jj = 0;
    for (int64_t item = s_item[0]; item < f.items;) {
      bool isb;
      int64_t ch;
      decode_item(f, item, isb, ch);
      if (!isb)
        run(A, pa, tAA, s_ba_u, ch);
      else
        run(B, pb, tAB, s_bb_u, ch);
      ++jj;
      item = s_item[jj & 1];
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc<COLS>(tbase);
}

}  // namespace tcfft
