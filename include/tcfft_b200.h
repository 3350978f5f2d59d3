/*
 * tcfft_b200.h - C ABI of the B200-native tcFFT (batched FP16 complex-to-complex
 * forward FFT on sm_100a tensor cores).
 *
 * The entry points are the cuFFT-style plan/execute surface the tcFFT paper
 * names and the reference package exposes in Python:
 *
 *   tcfftPlan1D   <- reference plan_1d(nx, batch)        pkg/src/tcfft/plan.py:116-122
 *   tcfftPlan2D   <- reference plan_2d(nx, ny, batch)    pkg/src/tcfft/plan.py:125-138
 *   tcfftExecC2C  <- reference execute(plan, data)       pkg/src/tcfft/executor.py:152-190
 *   tcfftDestroy  <- (garbage collection of Plan)        pkg/src/tcfft/plan.py:57
 *
 * Data layout: interleaved fp16 (re, im) pairs (cuFFT CUDA_C_16F), i.e. the
 * reference BatchedTensor pairs array (executor.py:25-51) in device memory,
 * contiguous: 1D element j of sequence b at [b*nx + j]; 2D row-major (nx, ny)
 * with ny contiguous.  The transform is forward (W = exp(-2*pi*i/N)),
 * unnormalised, natural order in and out, and may run in place
 * (odata == idata).  Errors map onto the reference's exception classes in the
 * Python wrapper (UnsupportedSizeError, PlanArgumentError, ExecuteError).
 * Plain pointers and sizes only: no framework types cross this boundary.
 */
#ifndef TCFFT_B200_H_
#define TCFFT_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tcfftPlanImpl* tcfftHandle;

typedef enum tcfftResult_t {
  TCFFT_SUCCESS = 0,
  TCFFT_INVALID_PLAN = 1,  /* null / destroyed handle */
  TCFFT_ALLOC_FAILED = 2,  /* device or host allocation failed */
  TCFFT_INVALID_VALUE = 3, /* bad argument (batch < 1, null pointer, misaligned buffer) */
  TCFFT_INVALID_SIZE = 4,  /* transform size not a power of two >= 2 */
  TCFFT_EXEC_FAILED = 5,   /* kernel launch / CUDA runtime failure */
  TCFFT_NOT_SUPPORTED = 6, /* valid size this build does not implement */
  TCFFT_NO_DEVICE = 7      /* no sm_100 device available */
} tcfftResult;

/* Plan a batch of 1D transforms of length nx (reference plan.py:116). */
tcfftResult tcfftPlan1D(tcfftHandle* plan, int nx, int batch);
/* Plan a batch of 2D transforms over row-major (nx, ny) data (plan.py:125). */
tcfftResult tcfftPlan2D(tcfftHandle* plan, int nx, int ny, int batch);
/* Stream for subsequent executions (cudaStream_t passed as void*; NULL = legacy default). */
tcfftResult tcfftSetStream(tcfftHandle plan, void* stream);
/* Concurrency: executions are ordered on the plan's stream.  tcfftExecC2C on
 * a plan without a workspace (tcfftGetWorkspaceSize == 0: 1D N <= 16384 and
 * all 2D plans) may run on several streams concurrently (different buffers;
 * set the stream and execute under one host lock).  Plans with a workspace
 * (1D N > 16384), tcfftExecC2CHost and the scratch path of
 * tcfftExecC2CStrided use plan-owned device memory and run one execution at a
 * time: use one plan per stream for those.  Every exec entry point returns
 * TCFFT_INVALID_VALUE when the calling thread's current device is not the
 * device the plan was created on. */
/* Bytes of device workspace the plan owns (0 for single-pass plans). */
tcfftResult tcfftGetWorkspaceSize(tcfftHandle plan, size_t* bytes);
/* Forward FP16 C2C transform; idata/odata are device pointers to __half2
 * (interleaved complex), 16-byte aligned; odata may equal idata. Asynchronous
 * with respect to the host (stream-ordered). */
tcfftResult tcfftExecC2C(tcfftHandle plan, const void* idata, void* odata);
/* Same transform with HOST buffers (the reference's execute() works on host
 * numpy data, executor.py:152): the batch is sliced and H2D copy, transform and
 * D2H copy of successive slices are pipelined on three internal streams.
 * hin/hout should be pinned (cudaHostAlloc / cudaHostRegister) for overlap;
 * may alias.  Ordered after prior work on the plan's stream; completion is
 * ordered before later work on it (synchronize the stream before reading hout). */
tcfftResult tcfftExecC2CHost(tcfftHandle plan, const void* hin, void* hout);
/* Strided views (reference BatchedTensor, executor.py:25-51): element j of
 * transform b at idata[b*batch_stride + j*stride] (complex elements), same for
 * odata; 2D plans require stride 1.  Contiguous views and row-pitched 1D
 * views (stride 1, batch_stride a multiple of 4: one-pass plans and the
 * two-pass plans of 2^15 .. 2^22) run the transform directly on the view;
 * other views go through a plan-owned contiguous scratch. */
tcfftResult tcfftExecC2CStrided(tcfftHandle plan, const void* idata, void* odata, long long stride,
                                long long batch_stride);
tcfftResult tcfftDestroy(tcfftHandle plan);
/* Profiling hook (not part of the reference interface): subsequent
 * tcfftExecC2C calls launch only the passes whose bit is set in `mask`
 * (bit i = pass i; ~0u restores normal execution).  Buffer routing is
 * unchanged, so a partial execution does NOT produce a transform; used by
 * bench.py to time each pass kernel on its own with CUDA events. */
tcfftResult tcfftSetPassMask(tcfftHandle plan, unsigned mask);

const char* tcfftGetErrorString(tcfftResult r);
int tcfftGetVersion(void);

/* ---- introspection (host-only, no GPU needed) --------------------------
 * tcfftDescribePlan writes a JSON description of the plan that tcfftPlan1D /
 * tcfftPlan2D would build (passes, radices, chunking, smem/TMEM budget).
 * tcfftPlanTables copies the per-pass host tables (row records, B matrices,
 * twiddle tables) so CPU tests can emulate the kernel's dataflow exactly.
 * Pass the null pointer to query the byte sizes. */
tcfftResult tcfftDescribePlan(int dims, int nx, int ny, int batch, char* json, size_t cap);
tcfftResult tcfftPlanTables(int dims, int nx, int ny, int batch, int pass, void* rows, size_t* rows_bytes,
                            void* bmats, size_t* b_bytes, void* twid, size_t* t_bytes);

/* ---- distributed single transforms (the reference has
 * no counterpart: SPEC.md:14,467 and PAPER.md:619 leave multi-GPU transforms
 * out of scope).  One 1D transform of length nx split over `world` ranks
 * (one process per GPU), four-step N = N1 N2 (N1 = 2^floor(log2(nx)/2)):
 *   rank g input  : column slab [N1][N2/world], x[N2 n1 + n2], n2 in block g
 *   pass 0        : tcfftExecDistPass(plan, 0, slab, slab)   column FFTs + twiddle
 *   exchange      : all-to-all of the slab's N1/world-row blocks (caller, NCCL)
 *   unpack        : tcfftDistUnpack(plan, world, recv, rows)  -> rows [N1/world][N2]
 *   pass 1        : tcfftExecDistPass(plan, 1, rows, out)     row FFTs, transposed
 *   rank g output : [N2][N1/world] = X[k1 + N1 k2], k1 in block g
 * N1, N2 <= 4096 and divisible by world (N <= 2^24).  Stream-ordered on the
 * plan's stream like tcfftExecC2C. */
tcfftResult tcfftPlan1DDist(tcfftHandle* plan, int nx, int rank, int world);
tcfftResult tcfftExecDistPass(tcfftHandle plan, int pass, const void* idata, void* odata);
tcfftResult tcfftDistUnpack(tcfftHandle plan, int world, const void* recv, void* rows);
/* Fused exchange (world <= 8): pass 0 stores each N1/world-row slice of its
 * tiles straight into the owning rank's receive buffer (peer memory over
 * NVLink / CUDA IPC mappings), blocked [N2/C][N1/world][C]; after a
 * cross-rank barrier pass 1 reads this rank's receive buffer:
 *   tcfftDistSetPeers(plan, recv, world)       recv[h] = rank h's receive buffer, mapped here
 *   tcfftExecDistPass(plan, 0, slab, slab)     compute + exchange
 *   (barrier)  tcfftExecDistPass(plan, 1, recv[rank], out)
 * tcfftIpc* wrap cudaIpcGetMemHandle / OpenMemHandle / CloseMemHandle
 * (handle = 64 opaque bytes) for processes that share the buffers. */
tcfftResult tcfftPlan1DDistFused(tcfftHandle* plan, int nx, int rank, int world);
tcfftResult tcfftDistSetPeers(tcfftHandle plan, const void* const* recv, int world);
tcfftResult tcfftIpcGetHandle(const void* dptr, void* handle, size_t cap);
tcfftResult tcfftIpcOpenHandle(const void* handle, void** dptr);
tcfftResult tcfftIpcCloseHandle(void* dptr);
tcfftResult tcfftDescribeDistPlan(int nx, int rank, int world, char* json, size_t cap);
tcfftResult tcfftDescribeDistPlanFused(int nx, int rank, int world, char* json, size_t cap);
tcfftResult tcfftDistPlanTablesFused(int nx, int rank, int world, int pass, void* rows, size_t* rows_bytes,
                                     void* bmats, size_t* b_bytes, void* twid, size_t* t_bytes);
tcfftResult tcfftDistPlanTables(int nx, int rank, int world, int pass, void* rows, size_t* rows_bytes, void* bmats,
                                size_t* b_bytes, void* twid, size_t* t_bytes);

#ifdef __cplusplus
}
#endif

#endif /* TCFFT_B200_H_ */
