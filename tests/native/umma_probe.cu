// umma_probe.cu - hardware check of the tcgen05 operand layouts the FFT
// kernels rely on (test infrastructure; run via tests/test_gpu_probe.py).
// Each variant computes D(128x32) = A(128x32) . B(32x32) with small-integer
// fp16 data (exact in fp32) and compares with a host GEMM.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>
#include "../../paper_2104_11471_b200/csrc/sm100.cuh"

using namespace sm100;
constexpr int M = 128, N = 32, K = 32;

struct Variant {
  const char* name;
  int ts;            // A from TMEM
  int a_mn;          // A MN-major
  uint32_t a_lbo, a_sbo, a_qstep;  // descriptor fields, per-K16-slice start step (bytes)
  uint32_t b_lbo, b_sbo, b_qstep;
};

__global__ void probe_kernel(const __half* A, const __half* B, const int* offA, const int* offB, Variant v,
                             float* D) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;            // 16 KB
  uint8_t* sB = smem + 16384;    // 8 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int t = threadIdx.x, warp = t / 32;
  for (int i = t; i < M * K; i += 128) *reinterpret_cast<__half*>(sA + offA[i]) = A[i];
  for (int i = t; i < K * N; i += 128) *reinterpret_cast<__half*>(sB + offB[i]) = B[i];
  if (warp == 0) tmem_alloc<64>(&tbase);
  if (t == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  uint32_t tm = tbase;
  uint32_t tA = tm + 32, tD = tm;  // columns 32..47 hold A (TS), 0..31 hold D
  if (v.ts) {
    uint32_t r[16];
    for (int c = 0; c < 16; ++c) {
      __half lo = A[t * K + 2 * c], hi = A[t * K + 2 * c + 1];
      r[c] = (uint32_t)__half_as_ushort(lo) | ((uint32_t)__half_as_ushort(hi) << 16);
    }
    tmem_st16(tA + ((uint32_t)(warp * 32) << 16), r);
    tmem_wait_st();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  if (t == 0) {
    tc_fence_after();
    uint32_t idesc = make_idesc_f16(M, N, v.a_mn, 0);
    for (int q = 0; q < K / 16; ++q) {
      uint64_t bd = make_sdesc(smem_u32(sB) + q * v.b_qstep, v.b_lbo, v.b_sbo);
      if (v.ts) {
        mma_ts(tD, tA + q * 8, bd, idesc, q > 0);
      } else {
        uint64_t ad = make_sdesc(smem_u32(sA) + q * v.a_qstep, v.a_lbo, v.a_sbo);
        mma_ss(tD, ad, bd, idesc, q > 0);
      }
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[32];
  tmem_ld32(tD + ((uint32_t)(warp * 32) << 16), r);
  tmem_wait_ld();
  for (int n = 0; n < 32; ++n) D[t * N + n] = __uint_as_float(r[n]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<64>(tm);
}

__global__ void math_kernel(float* out) {
  float2 a = make_float2(1.5f, -2.0f), b = make_float2(3.0f, 0.25f), c = make_float2(0.5f, 1.0f);
  float2 d = ffma2(a, b, c);
  float2 e = fmul2(a, b);
  out[0] = d.x; out[1] = d.y; out[2] = e.x; out[3] = e.y;
  uint32_t p = pack_half2(1.0f, -2.0f);
  out[4] = __half2float(__ushort_as_half(p & 0xffff));
  out[5] = __half2float(__ushort_as_half(p >> 16));
}

static int offK(int row, int k, int lbo, int sbo) { return (row % 8) * 16 + (row / 8) * sbo + (k / 8) * lbo + (k % 8) * 2; }
static int offMN(int m, int k, int lbo, int sbo) { return (m % 8) * 2 + (m / 8) * sbo + (k / 8) * lbo + (k % 8) * 16; }

int main() {
  std::vector<__half> hA(M * K), hB(K * N);
  std::vector<float> fA(M * K), fB(K * N), ref(M * N);
  srand(1234);
  for (int i = 0; i < M * K; ++i) { fA[i] = (float)(rand() % 9 - 4); hA[i] = __float2half(fA[i]); }
  for (int i = 0; i < K * N; ++i) { fB[i] = (float)(rand() % 9 - 4); hB[i] = __float2half(fB[i]); }
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += fA[m * K + k] * fB[k * N + n];
      ref[m * N + n] = (float)s;
    }
  // B stored K-major (per output column n, K contiguous): element (k, n).
  Variant vs[] = {
      {"SS A-Kmajor", 0, 0, 128, 512, 256, 128, 512, 256},
      {"SS A-MNmajor sbo=528", 0, 1, 128, 528, 256, 128, 512, 256},
      {"SS A-MNmajor sbo=512", 0, 1, 128, 512, 256, 128, 512, 256},
      {"SS A-MNmajor swapped(lbo=528,sbo=128)", 0, 1, 528, 128, 256, 128, 512, 256},
      {"TS A-tmem", 1, 0, 0, 0, 0, 128, 512, 256},
  };
  __half *dA, *dB; int *dOA, *dOB; float* dD;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, K * N * 2); cudaMalloc(&dOA, M * K * 4); cudaMalloc(&dOB, K * N * 4);
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), K * N * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  int fails = 0;
  for (auto& v : vs) {
    std::vector<int> oA(M * K), oB(K * N);
    int a_sbo = (v.a_mn && v.a_lbo == 528) ? 528 : v.a_sbo;  // layout follows the intended SBO
    for (int m = 0; m < M; ++m)
      for (int k = 0; k < K; ++k)
        oA[m * K + k] = v.a_mn ? offMN(m, k, 128, (v.a_lbo == 528 ? 528 : v.a_sbo)) : offK(m, k, 128, 512);
    (void)a_sbo;
    for (int k = 0; k < K; ++k)
      for (int n = 0; n < N; ++n) oB[k * N + n] = offK(n, k, 128, 512);
    cudaMemcpy(dOA, oA.data(), M * K * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dOB, oB.data(), K * N * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, M * N * 4);
    probe_kernel<<<1, 128, 32768>>>(dA, dB, dOA, dOB, v, dD);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> got(M * N);
    cudaMemcpy(got.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
    double err = 0, errT = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) err = fmax(err, fabs(got[m * N + n] - ref[m * N + n]));
    printf("PROBE %-40s cuda=%s maxerr=%g  d[0][0..3]=%g %g %g %g ref=%g %g %g %g\n", v.name, cudaGetErrorString(e),
           err, got[0], got[1], got[2], got[3], ref[0], ref[1], ref[2], ref[3]);
    (void)errT;
    if (e != cudaSuccess) return 2;
  }
  float* dm; cudaMalloc(&dm, 64);
  math_kernel<<<1, 1>>>(dm);
  float hm[6]; cudaMemcpy(hm, dm, 24, cudaMemcpyDeviceToHost);
  printf("MATH ffma2=(%g,%g) want (5,0.5); fmul2=(%g,%g) want (4.5,-0.5); pack=(%g,%g) want (1,-2)\n", hm[0], hm[1],
         hm[2], hm[3], hm[4], hm[5]);
  return fails;
}
