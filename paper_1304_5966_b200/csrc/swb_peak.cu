// Integer / DPX instruction-throughput microbenchmark for the cell-update roofline.
//
// The SW# cell update is a max-plus recurrence executed on the
// integer pipes, so the roofline denominator is the chip's sustained issue rate of
// the instructions the recurrence lowers to (VIADDMNMX, VIMNMX3, PRMT, IADD3).
// Each kernel below runs NCHAIN independent dependency chains per thread so the
// measurement is throughput-bound, not latency-bound.  The C-ABI entry point
// swb_measure_int_peak() (include/swb.h) returns warp-lane ops per second for each
// instruction class, measured with CUDA events on the launching stream.
#include <cuda_runtime.h>
#include <stdint.h>
#include "swb_internal.h"

namespace {

constexpr int NCHAIN = 8;

template <int KIND>
__global__ void __launch_bounds__(256) peak_kernel(int iters, int seed, int* sink) {
  int v[NCHAIN];
#pragma unroll
  for (int k = 0; k < NCHAIN; ++k) v[k] = seed * (k + 1) + threadIdx.x;
  const int b = seed ^ 0x5a5a;
  const int c = seed - 77;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < NCHAIN; ++k) {
        if (KIND == 0) {          // VIADDMNMX: max(a + b, c)
          v[k] = __viaddmax_s32(v[k], b, c + k);
        } else if (KIND == 1) {   // VIMNMX3: max(a, b, c)
          v[k] = __vimax3_s32(v[k], b + k, c);
        } else if (KIND == 2) {   // VIADDMNMX.RELU
          v[k] = __viaddmax_s32_relu(v[k], b, c + k);
        } else if (KIND == 3) {   // IADD (Fibonacci pairs: no closed form to fold)
          v[k] = v[k] + v[(k + 1) % NCHAIN];
        } else if (KIND == 4) {   // PRMT
          v[k] = __byte_perm(v[k], b, 0x8880 + k);
        } else if (KIND == 5) {   // IMAD (fma pipe)
          v[k] = v[k] * (b | 1) + v[(k + 1) % NCHAIN];
        }
      }
    }
  }
  int acc = 0;
#pragma unroll
  for (int k = 0; k < NCHAIN; ++k) acc ^= v[k];
  if (acc == 0x7fffffff) sink[blockIdx.x] = acc;  // keep the chains live
}

template <int KIND>
double run_kind(cudaStream_t st, int* sink, int blocks, int iters, float* ms_out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  peak_kernel<KIND><<<blocks, 256, 0, st>>>(2, 3, sink);  // warm-up
  cudaEventRecord(e0, st);
  peak_kernel<KIND><<<blocks, 256, 0, st>>>(iters, 3, sink);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *ms_out = ms;
  double ops = (double)blocks * 256.0 * (double)iters * 16.0 * NCHAIN;
  return ops / (ms * 1e-3);
}

}  // namespace

extern "C" int swb_measure_int_peak(swb_ctx* ctx, swb_int_peak* out) {
  SWB_API_BEGIN(ctx);
  int dev = ctx->device;
  int sms = 0;
  SWB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int* sink = nullptr;
  SWB_CUDA(cudaMalloc(&sink, sizeof(int) * 65536));
  const int blocks = sms * 8;  // 8 x 256 threads = 64 warps per SM
  const int iters = 4096;
  cudaStream_t st = ctx->stream;
  float ms = 0.f;
  out->viaddmnmx = run_kind<0>(st, sink, blocks, iters, &ms);
  out->vimnmx3 = run_kind<1>(st, sink, blocks, iters, &ms);
  out->viaddmnmx_relu = run_kind<2>(st, sink, blocks, iters, &ms);
  out->iadd = run_kind<3>(st, sink, blocks, iters, &ms);
  out->prmt = run_kind<4>(st, sink, blocks, iters, &ms);
  out->imad = run_kind<5>(st, sink, blocks, iters, &ms);
  out->ms_last = ms;
  out->sms = sms;
  SWB_CUDA(cudaGetLastError());
  SWB_CUDA(cudaStreamSynchronize(st));
  cudaFree(sink);
  SWB_API_END();
}
