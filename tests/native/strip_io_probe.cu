// strip_io_probe.cu - data-movement ceiling of a column-strip pass (probe, not
// product code).  Copies a [B][L][W] array of 4-byte elements strip by strip
// (C columns x L rows per chunk) with the same TMA 3D boxes the FFT strip pass
// uses, and, for comparison, with plain 16-byte LSU loads/stores.  Reports
// GB/s (read + write) so that the FFT pass's roofline fraction can be compared
// with what the access pattern alone achieves.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o strip_io_probe strip_io_probe.cu -lcuda
//   ./strip_io_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
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

struct P {
  int L, W, C, spi, nsub, boxr, bufs;
  long long chunks;
};

__global__ void __launch_bounds__(128) tma_strip_copy(const __grid_constant__ CUtensorMap tin,
                                                      const __grid_constant__ CUtensorMap tout, P p) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar[4];
  const int bytes = p.L * p.C * 4;
  if (threadIdx.x == 0) {
    for (int i = 0; i < p.bufs; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t phase = 0;
  auto load = [&](long long ch, int b) {
    uint8_t* dst = sm + b * bytes;
    const int img = (int)(ch / p.spi), cb = (int)(ch % p.spi);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[b])), "r"(bytes));
    for (int i = 0; i < p.nsub; ++i)
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(su32(dst + i * p.boxr * p.C * 4)),
          "l"(&tin), "r"(cb * p.C), "r"(i * p.boxr), "r"(img), "r"(su32(&bar[b]))
          : "memory");
  };
  auto store = [&](long long ch, int b) {
    const uint8_t* src = sm + b * bytes;
    const int img = (int)(ch / p.spi), cb = (int)(ch % p.spi);
    for (int i = 0; i < p.nsub; ++i)
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&tout),
                   "r"(cb * p.C), "r"(i * p.boxr), "r"(img), "r"(su32(src + i * p.boxr * p.C * 4))
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  };
  // ring of `bufs` staging buffers: load k+bufs-1 ahead
  const long long n = (p.chunks - blockIdx.x + gridDim.x - 1) / gridDim.x;
  auto mine = [&](long long i) { return (long long)blockIdx.x + i * gridDim.x; };
  for (int i = 0; i < p.bufs - 1 && i < n; ++i) load(mine(i), i);
  for (long long i = 0; i < n; ++i) {
    const int b = (int)(i % p.bufs);
    const int nb = (int)((i + p.bufs - 1) % p.bufs);
    if (i + p.bufs - 1 < n) {
      // buffer nb was last stored at iteration i-1: wait until that store read it
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      load(mine(i + p.bufs - 1), nb);
    }
    const uint32_t par = (phase >> b) & 1;
    asm volatile(
        "{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
            su32(&bar[b])),
        "r"(par)
        : "memory");
    phase ^= 1u << b;
    store(mine(i), b);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// LSU: each thread moves 16 B rows (C = 4 words) of a strip, 1 row per thread per step
__global__ void lsu_strip_copy(const uint4* __restrict__ in, uint4* __restrict__ out, P p) {
  const long long rows_total = p.chunks * p.L;  // chunk-major rows
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < rows_total;
       r += (long long)gridDim.x * blockDim.x) {
    const long long ch = r / p.L;
    const int row = (int)(r % p.L);
    const long long img = ch / p.spi, cb = ch % p.spi;
    const long long off = (img * p.L + row) * (long long)(p.W / 4) + cb * (p.C / 4);
#pragma unroll
    for (int q = 0; q < p.C / 4; ++q) out[off + q] = in[off + q];
  }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncFn enc() {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
  return (EncFn)f;
}

int main() {
  const long long total = 1ll << 28;  // 1 GiB of 4-byte elements, like C3 / C4
  uint32_t *a, *b;
  CK(cudaMalloc(&a, total * 4));
  CK(cudaMalloc(&b, total * 4));
  CK(cudaMemset(a, 1, total * 4));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(tma_strip_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
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
  // plain copy reference
  float ms = time_it([&] { cudaMemcpyAsync(b, a, total * 4, cudaMemcpyDeviceToDevice); });
  std::printf("{\"probe\": \"memcpy\", \"gbs\": %.1f}\n", total * 8 / (ms * 1e-3) / 1e9);
  struct Case {
    int L, W, C, ctas, bufs;
    long long elems;  // working set (4-byte elements); 2^23 = 32 MiB in + 32 MiB out stays in L2
    int prom;         // TMA L2 promotion: 0 none, 256 = 256B
  };
  const long long G = 1ll << 28, S = 1ll << 23;
  std::vector<Case> cases = {
      {2048, 2048, 4, 2, 1, G, 256}, {2048, 2048, 4, 2, 1, G, 0},   {2048, 2048, 4, 2, 1, S, 256},
      {2048, 2048, 4, 4, 1, S, 256}, {2048, 2048, 8, 2, 1, G, 256}, {2048, 2048, 8, 2, 2, G, 256},
      {2048, 2048, 8, 2, 2, S, 256}, {2048, 2048, 16, 1, 1, G, 256}, {2048, 2048, 16, 1, 1, S, 256},
      {1024, 1024, 8, 4, 1, G, 256}, {1024, 1024, 8, 4, 1, S, 256}, {512, 512, 8, 4, 1, G, 256},
      {512, 512, 8, 4, 1, S, 256},   {256, 16384, 16, 4, 1, G, 256}, {256, 16384, 32, 2, 1, G, 256},
      {512, 8192, 16, 2, 1, G, 256}, {512, 8192, 8, 4, 1, G, 256},  {256, 256, 16, 4, 1, S, 256},
  };
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
    const long long imgs = c.elems / ((long long)c.L * c.W);
    p.chunks = imgs * p.spi;
    CUtensorMap ti, to;
    cuuint64_t dims[3] = {(cuuint64_t)c.W, (cuuint64_t)c.L, (cuuint64_t)imgs};
    cuuint64_t strides[2] = {(cuuint64_t)c.W * 4, (cuuint64_t)c.W * c.L * 4};
    cuuint32_t box[3] = {(cuuint32_t)c.C, (cuuint32_t)p.boxr, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CK(E(&ti, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, a, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, c.prom ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    CK(E(&to, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, b, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    const int smem = c.bufs * c.L * c.C * 4;
    long long grid = (long long)sms * c.ctas;
    if (grid > p.chunks) grid = p.chunks;
    ms = time_it([&] { tma_strip_copy<<<(int)grid, 128, smem>>>(ti, to, p); });
    CK(cudaGetLastError());
    std::printf("{\"probe\": \"tma\", \"L\": %d, \"W\": %d, \"C\": %d, \"run_bytes\": %d, \"ctas_per_sm\": %d, "
                "\"bufs\": %d, \"chunk_kib\": %d, \"mib\": %lld, \"prom\": %d, \"gbs\": %.1f}\n",
                c.L, c.W, c.C, c.C * 4, c.ctas, c.bufs, c.L * c.C * 4 / 1024, c.elems * 4 >> 20, c.prom,
                c.elems * 8 / (ms * 1e-3) / 1e9);
    if (c.bufs == 1 && c.ctas <= 2 && c.C == 4) {
      ms = time_it([&] { lsu_strip_copy<<<sms * 16, 256>>>((const uint4*)a, (uint4*)b, p); });
      std::printf("{\"probe\": \"lsu\", \"L\": %d, \"W\": %d, \"C\": %d, \"run_bytes\": %d, \"gbs\": %.1f}\n", c.L,
                  c.W, c.C, c.C * 4, c.elems * 8 / (ms * 1e-3) / 1e9);
    }
  }
  return 0;
}
