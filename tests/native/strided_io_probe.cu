// strided_io_probe.cu - data-movement ceilings of the strided sides of the
// multi-pass plans (probe, not product code).
//
// A [B][L][W] array of 4-byte elements is moved chunk by chunk, a chunk being
// a strip of C columns x L rows (what a column / four-step pass holds in
// shared memory).  Each side is done one of three ways:
//   read : tma  = 3D TMA boxes {C, 256, 1} (the FFT passes' strided loads)
//          cpa  = cp.async.cg 16-byte copies issued by all 128 threads,
//                 completion tracked by the same mbarrier (noinc arrive)
//          lin  = the chunk's bytes as one contiguous bulk copy (blocked layout)
//   write: tma  = 3D TMA boxes (strided), stg = 16-byte st.global by all
//          threads (strided), lin = one contiguous bulk copy
// Pass 1 of the two-pass 1D plan is read=strided / write=lin, pass 2 is
// read=lin / write=strided, a 2D column pass is strided / strided.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o strided_io_probe strided_io_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                    \
  do {                                                                           \
    auto e_ = (x);                                                               \
    if (e_ != 0) {                                                               \
      std::printf("error %d at %s:%d\n", (int)e_, __FILE__, __LINE__);           \
      std::exit(1);                                                              \
    }                                                                            \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

enum { RD_TMA = 0, RD_CPA = 1, RD_LIN = 2 };
enum { WR_TMA = 0, WR_STG = 1, WR_LIN = 2 };

struct P {
  int L, W, C, spi, nsub, boxr, bufs, rd, wr;
  long long chunks;
  const uint8_t* gin;
  uint8_t* gout;
};

__device__ __forceinline__ void mwait(uint64_t* bar, uint32_t par) {
  asm volatile(
      "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(su32(bar)),
      "r"(par)
      : "memory");
}

__global__ void __launch_bounds__(128) strided_copy(const __grid_constant__ CUtensorMap tin,
                                                    const __grid_constant__ CUtensorMap tout, P p) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[4];
  const int bytes = p.L * p.C * 4;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < p.bufs; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[i])), "r"(p.rd == RD_CPA ? 129 : 1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int pieces_row = p.C / 4;  // 16-byte pieces per strip row
  const int pieces = p.L * pieces_row;
  auto goff = [&](long long ch, int row) -> long long {  // byte offset of (chunk, row, column 0)
    const long long img = ch / p.spi, cb = ch % p.spi;
    return ((img * p.L + row) * (long long)p.W + cb * p.C) * 4;
  };
  // every thread calls load(); only the issuing threads do work
  auto load = [&](long long ch, int b) {
    uint8_t* dst = sm + b * bytes;
    if (p.rd == RD_CPA) {
      if (tid == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[b])), "r"(0));
      for (int q = tid; q < pieces; q += 128) {
        const int row = q / pieces_row, c = q % pieces_row;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + q * 16)),
                     "l"(p.gin + goff(ch, row) + c * 16)
                     : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&bar[b])) : "memory");
      return;
    }
    if (tid != 0) return;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[b])), "r"(bytes));
    if (p.rd == RD_LIN) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       su32(dst)),
                   "l"(p.gin + ch * (long long)bytes), "r"(bytes), "r"(su32(&bar[b]))
                   : "memory");
      return;
    }
    const int img = (int)(ch / p.spi), cb = (int)(ch % p.spi);
    for (int i = 0; i < p.nsub; ++i)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(su32(dst + i * p.boxr * p.C * 4)),
          "l"(&tin), "r"(cb * p.C), "r"(i * p.boxr), "r"(img), "r"(su32(&bar[b]))
          : "memory");
  };
  auto store = [&](long long ch, int b) {
    const uint8_t* src = sm + b * bytes;
    if (p.wr == WR_STG) {
      for (int q = tid; q < pieces; q += 128) {
        const int row = q / pieces_row, c = q % pieces_row;
        uint4 v;
        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                     : "r"(su32(src + q * 16)));
        *reinterpret_cast<uint4*>(p.gout + goff(ch, row) + c * 16) = v;
      }
      return;
    }
    if (tid != 0) return;
    if (p.wr == WR_LIN) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p.gout + ch * (long long)bytes),
                   "r"(su32(src)), "r"(bytes)
                   : "memory");
    } else {
      const int img = (int)(ch / p.spi), cb = (int)(ch % p.spi);
      for (int i = 0; i < p.nsub; ++i)
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&tout),
                     "r"(cb * p.C), "r"(i * p.boxr), "r"(img), "r"(su32(src + i * p.boxr * p.C * 4))
                     : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  };
  const long long n = (p.chunks - blockIdx.x + gridDim.x - 1) / gridDim.x;
  auto mine = [&](long long i) { return (long long)blockIdx.x + i * gridDim.x; };
  for (int i = 0; i < p.bufs - 1 && i < n; ++i) load(mine(i), i);
  uint32_t phase = 0;
  for (long long i = 0; i < n; ++i) {
    const int b = (int)(i % p.bufs);
    const int nb = (int)((i + p.bufs - 1) % p.bufs);
    if (i + p.bufs - 1 < n) {
      // buffer nb was last stored at iteration i-1: wait until that store has read it
      if (p.wr != WR_STG) {
        if (tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
      __syncthreads();
      load(mine(i + p.bufs - 1), nb);
    }
    mwait(&bar[b], (phase >> b) & 1);
    phase ^= 1u << b;
    if (p.wr != WR_STG) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    store(mine(i), b);
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncFn enc() {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
  return (EncFn)f;
}

int main() {
  const long long total = 1ll << 28;  // 1 GiB of 4-byte elements, like C3 / C4
  uint8_t *a, *b;
  CK(cudaMalloc(&a, total * 4));
  CK(cudaMalloc(&b, total * 4));
  CK(cudaMemset(a, 1, total * 4));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  CK(cudaFuncSetAttribute(strided_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 225 * 1024));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time_it = [&](auto fn) {
    fn();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      fn();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    return best;
  };
  float ms = time_it([&] { cudaMemcpyAsync(b, a, total * 4, cudaMemcpyDeviceToDevice); });
  std::printf("{\"probe\": \"memcpy\", \"gbs\": %.1f}\n", total * 8 / (ms * 1e-3) / 1e9);
  const char* rn[] = {"tma", "cpa", "lin"};
  const char* wn[] = {"tma", "stg", "lin"};
  struct Case {
    int L, W, C, ctas, bufs, rd, wr;
  };
  std::vector<Case> cases;
  // C3 two-pass (2048 x 2048) and 2D 2048^2 / 4096^2 column geometries
  for (int geo = 0; geo < 2; ++geo) {
    const int L = geo == 0 ? 2048 : 4096, W = L;
    for (int C : {4, 8, 16}) {
      const int kb = L * C * 4 / 1024;
      for (int ctas : {1, 2, 4})
        for (int bufs : {1, 2}) {
          if (ctas * bufs * kb > 220) continue;
          for (int rd : {RD_TMA, RD_CPA}) cases.push_back({L, W, C, ctas, bufs, rd, WR_LIN});  // pass 1
          for (int wr : {WR_TMA, WR_STG}) cases.push_back({L, W, C, ctas, bufs, RD_LIN, wr});  // pass 2
          if (geo == 1 || C == 8)
            for (int rd : {RD_TMA, RD_CPA})
              for (int wr : {WR_TMA, WR_STG}) cases.push_back({L, W, C, ctas, bufs, rd, wr});  // 2D columns
        }
    }
  }
  auto E = enc();
  for (auto c : cases) {
    P p;
    p.L = c.L;
    p.W = c.W;
    p.C = c.C;
    p.spi = c.W / c.C;
    p.boxr = c.L < 256 ? c.L : 256;
    p.nsub = c.L / p.boxr;
    p.bufs = c.bufs;
    p.rd = c.rd;
    p.wr = c.wr;
    p.gin = a;
    p.gout = b;
    const long long imgs = total / ((long long)c.L * c.W);
    p.chunks = imgs * p.spi;
    CUtensorMap ti, to;
    cuuint64_t dims[3] = {(cuuint64_t)c.W, (cuuint64_t)c.L, (cuuint64_t)imgs};
    cuuint64_t strides[2] = {(cuuint64_t)c.W * 4, (cuuint64_t)c.W * c.L * 4};
    cuuint32_t box[3] = {(cuuint32_t)c.C, (cuuint32_t)p.boxr, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CK(E(&ti, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, a, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    CK(E(&to, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, b, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    const int smem = c.bufs * c.L * c.C * 4;
    long long grid = (long long)sms * c.ctas;
    if (grid > p.chunks) grid = p.chunks;
    ms = time_it([&] { strided_copy<<<(int)grid, 128, smem>>>(ti, to, p); });
    CK(cudaGetLastError());
    std::printf("{\"L\": %d, \"C\": %d, \"run_bytes\": %d, \"ctas_per_sm\": %d, \"bufs\": %d, \"read\": \"%s\", "
                "\"write\": \"%s\", \"chunk_kib\": %d, \"gbs\": %.1f}\n",
                c.L, c.C, c.C * 4, c.ctas, c.bufs, rn[c.rd], wn[c.wr], c.L * c.C * 4 / 1024,
                total * 8 / (ms * 1e-3) / 1e9);
  }
  return 0;
}
