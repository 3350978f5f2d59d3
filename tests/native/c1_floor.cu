// c1_floor.cu - latency floor of the C1 workload (probe, not product code).
//
// C1 moves 4 MiB in + 4 MiB out per launch (1D N=256 x 4096, fp16 pairs).
// bench.py times it as a CUDA graph of 64 launches over 64 rotating buffer
// pairs (512 MiB per cycle, so every launch misses L2).  This probe times,
// under exactly those conditions, what a launch costs with no FFT work:
//   empty   : an empty kernel with the C1 launch shape (512 CTAs x 128 threads)
//   tma<E>  : one bulk TMA load (E*4 bytes) -> mbarrier -> one bulk TMA store
//             per CTA, E = 1024 / 2048 / 4096 complex elements per CTA
//   memcpy  : cudaMemcpyAsync device-to-device of the same 4 MiB
// so that the FFT kernel's 4.8 us per launch can be compared with the floor.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o c1_floor c1_floor.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                \
  do {                                                                       \
    cudaError_t e_ = (x);                                                    \
    if (e_ != cudaSuccess) {                                                 \
      std::printf("cuda error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                          \
    }                                                                        \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128) empty_kernel(const uint8_t*, uint8_t*) {}

template <int BYTES>
__global__ void __launch_bounds__(128) tma_copy(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst) {
  __shared__ __align__(128) uint8_t buf[BYTES];
  __shared__ uint64_t bar;
  if (threadIdx.x != 0) return;
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t off = (size_t)blockIdx.x * BYTES;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(BYTES) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(buf)),
               "l"(src + off), "r"(BYTES), "r"(su32(&bar))
               : "memory");
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(su32(&bar))
        : "memory");
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off), "r"(su32(buf)),
               "r"(BYTES)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t bytes = 4u << 20;  // 4 MiB per direction (C1)
  const int nbuf = 64;
  std::vector<uint8_t*> in(nbuf), out(nbuf);
  for (int i = 0; i < nbuf; ++i) {
    CK(cudaMalloc(&in[i], bytes));
    CK(cudaMalloc(&out[i], bytes));
    CK(cudaMemset(in[i], 1, bytes));
  }
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  auto time_graph = [&](const char* name, auto launch) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < nbuf; ++i) launch(i);
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int w = 0; w < 5; ++w) CK(cudaGraphLaunch(ge, st));
    CK(cudaStreamSynchronize(st));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float best = 1e30f, sum = 0.f;
    const int reps = 20;
    for (int r = 0; r < reps; ++r) {
      CK(cudaEventRecord(e0, st));
      CK(cudaGraphLaunch(ge, st));
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      best = ms < best ? ms : best;
      sum += ms;
    }
    const double us = 1e3 * (sum / reps) / nbuf;
    std::printf("FLOOR %-8s us_per_launch=%.3f best=%.3f gbs=%.1f\n", name, us, 1e3 * best / nbuf,
                2.0 * bytes / (us * 1e-6) / 1e9);
    CK(cudaGraphExecDestroy(ge));
    CK(cudaGraphDestroy(g));
  };
  time_graph("empty", [&](int i) { empty_kernel<<<512, 128, 0, st>>>(in[i], out[i]); });
  time_graph("tma1024", [&](int i) { tma_copy<4096><<<(int)(bytes / 4096), 128, 0, st>>>(in[i], out[i]); });
  time_graph("tma2048", [&](int i) { tma_copy<8192><<<(int)(bytes / 8192), 128, 0, st>>>(in[i], out[i]); });
  time_graph("tma4096", [&](int i) { tma_copy<16384><<<(int)(bytes / 16384), 128, 0, st>>>(in[i], out[i]); });
  time_graph("memcpy", [&](int i) { CK(cudaMemcpyAsync(out[i], in[i], bytes, cudaMemcpyDeviceToDevice, st)); });
  return 0;
}
