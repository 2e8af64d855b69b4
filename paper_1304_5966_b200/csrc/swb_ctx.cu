// Context, error reporting, sequence upload and scratch management for libswb.so.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "swb_internal.h"

static thread_local char g_err[1024] = "";

void swb_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int swb_fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

// Scratch grows geometrically: a Myers-Miller level doubles its subproblem
// count, so a 25 % headroom would reallocate (cudaFree synchronises, pinned
// host allocation is slow) at every level of the first alignment.
static size_t grow_size(size_t bytes) {
  return bytes < ((size_t)256 << 20) ? 4 * bytes : bytes + bytes / 4;
}

void* swb_scratch(swb_buf& b, size_t bytes) {
  if (bytes == 0) bytes = 256;
  if (b.cap >= bytes) return b.p;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  size_t want = grow_size(bytes);
  if (cudaMalloc(&b.p, want) != cudaSuccess) {
    b.p = nullptr;
    cudaGetLastError();
    return nullptr;
  }
  b.cap = want;
  return b.p;
}

void* swb_scratch_host(swb_buf& b, size_t bytes) {
  if (bytes == 0) bytes = 256;
  if (b.cap >= bytes) return b.p;
  if (b.p) cudaFreeHost(b.p);
  b.p = nullptr;
  b.cap = 0;
  size_t want = grow_size(bytes);
  if (cudaMallocHost(&b.p, want) != cudaSuccess) {
    b.p = nullptr;
    cudaGetLastError();
    return nullptr;
  }
  b.cap = want;
  return b.p;
}

__global__ void reverse_kernel(const uint8_t* __restrict__ in, uint8_t* __restrict__ out, int64_t n) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
       x += (int64_t)gridDim.x * blockDim.x)
    out[n - 1 - x] = in[x];
}

extern "C" {

const char* swb_last_error(void) { return g_err; }

int32_t swb_version(void) { return 1; }

swb_ctx* swb_ctx_create(int32_t device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    swb_set_error("no CUDA device available: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return nullptr;
  }
  if (device < 0 || device >= count) {
    swb_set_error("device %d out of range (%d devices)", device, count);
    return nullptr;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    swb_set_error("cudaSetDevice(%d) failed", device);
    return nullptr;
  }
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  if (prop.major < 10) {
    swb_set_error("libswb.so is built for sm_100a; device %d is sm_%d%d", device, prop.major,
                  prop.minor);
    return nullptr;
  }
  swb_ctx* ctx = new swb_ctx();
  ctx->device = device;
  ctx->trace = getenv("SWB_TRACE") != nullptr;
  if (const char* w = getenv("SWB_WATCHDOG_MS")) ctx->watchdog_ms = atoi(w);
  if (getenv("SWB_CLAIM_LOG")) ctx->claim_log_on = 1;
  ctx->sms = prop.multiProcessorCount;
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess) {
    swb_set_error("stream/event creation failed");
    delete ctx;
    return nullptr;
  }
  return ctx;
}

void swb_ctx_destroy(swb_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& s : ctx->seqs) {
    if (s.fwd) cudaFree(s.fwd);
    if (s.rev) cudaFree(s.rev);
  }
  swb_buf* bufs[] = {&ctx->jobs,  &ctx->rowbuf, &ctx->progress, &ctx->results, &ctx->finals,
                     &ctx->misc,  &ctx->flush,  &ctx->bmap_fwd, &ctx->bmap_rev, &ctx->bmap_live,
                     &ctx->pass_finals, &ctx->dbg_buf, &ctx->claim_log, &ctx->wide_buf};
  if (ctx->tev0) {
    cudaEventDestroy(ctx->tev0);
    cudaEventDestroy(ctx->tev1);
  }
  for (auto* b : bufs)
    if (b->p) cudaFree(b->p);
  if (ctx->host_pinned.p) cudaFreeHost(ctx->host_pinned.p);
  cudaEventDestroy(ctx->ev0);
  cudaEventDestroy(ctx->ev1);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
}

int32_t swb_seq_upload(swb_ctx* ctx, const uint8_t* codes, int64_t n, int32_t* seq_id) {
  SWB_API_BEGIN(ctx);
  if (n < 0 || (n > 0 && codes == nullptr) || seq_id == nullptr)
    return swb_fail(SWB_EINVAL, "swb_seq_upload: bad arguments");
  if (n >= (int64_t)1 << 31) return swb_fail(SWB_ERANGE, "sequence longer than 2^31-1");
  {
    uint8_t acc = 0;
    for (int64_t x = 0; x < n; ++x) acc |= (uint8_t)(codes[x] >= 32);
    if (acc) {
      int64_t x = 0;
      while (codes[x] < 32) ++x;
      return swb_fail(SWB_EUNSUPPORTED,
                      "residue code %d at offset %lld: alphabets of more than 32 symbols are not supported",
                      (int)codes[x], (long long)x);
    }
  }
  // reuse a released slot whose device buffers are large enough (released
  // sequences keep their memory: no cudaMalloc/cudaFree per alignment call)
  int slot = -1;
  for (size_t k = 0; k < ctx->seqs.size(); ++k)
    if (!ctx->seqs[k].live && ctx->seqs[k].cap >= n && (slot < 0 || ctx->seqs[k].cap < ctx->seqs[slot].cap))
      slot = (int)k;
  if (slot < 0) {
    for (size_t k = 0; k < ctx->seqs.size(); ++k)
      if (!ctx->seqs[k].live) {
        slot = (int)k;
        break;
      }
    if (slot < 0) {
      ctx->seqs.push_back(swb_seq());
      slot = (int)ctx->seqs.size() - 1;
    }
    swb_seq& sq = ctx->seqs[slot];
    if (sq.fwd) cudaFree(sq.fwd);
    if (sq.rev) cudaFree(sq.rev);
    sq.fwd = sq.rev = nullptr;
    sq.cap = 0;
    const size_t bytes = n > 0 ? (size_t)n : 1;
    SWB_CUDA(cudaMalloc(&sq.fwd, bytes));
    SWB_CUDA(cudaMalloc(&sq.rev, bytes));
    sq.cap = (int64_t)bytes;
  }
  swb_seq& sq = ctx->seqs[slot];
  sq.n = n;
  {
    uint8_t c4 = 0;
    for (int64_t x = 0; x < n; ++x) c4 |= (uint8_t)(codes[x] == 4);
    sq.has_code4 = c4 != 0;
  }
  if (n > 0) {
    SWB_CUDA(cudaMemcpyAsync(sq.fwd, codes, (size_t)n, cudaMemcpyHostToDevice, ctx->stream));
    int blocks = (int)((n + 255) / 256);
    if (blocks > 4096) blocks = 4096;
    reverse_kernel<<<blocks, 256, 0, ctx->stream>>>(sq.fwd, sq.rev, n);
    ctx->launches++;
    SWB_CUDA(cudaGetLastError());
  }
  SWB_CUDA(cudaStreamSynchronize(ctx->stream));
  sq.live = true;
  *seq_id = (int32_t)slot;
  SWB_API_END();
}

int32_t swb_seq_release(swb_ctx* ctx, int32_t seq_id) {
  SWB_API_BEGIN(ctx);
  if (seq_id < 0 || seq_id >= (int32_t)ctx->seqs.size() || !ctx->seqs[seq_id].live)
    return swb_fail(SWB_EINVAL, "bad sequence id %d", seq_id);
  ctx->seqs[seq_id].live = false;  // memory kept for reuse (freed with the context)
  SWB_API_END();
}

double swb_last_kernel_ms(swb_ctx* ctx) { return ctx ? ctx->last_kernel_ms : 0.0; }

int32_t swb_timer_start(swb_ctx* ctx) {
  SWB_API_BEGIN(ctx);
  if (!ctx->tev0) {
    SWB_CUDA(cudaEventCreate(&ctx->tev0));
    SWB_CUDA(cudaEventCreate(&ctx->tev1));
  }
  SWB_CUDA(cudaEventRecord(ctx->tev0, ctx->stream));
  SWB_API_END();
}

int32_t swb_timer_stop(swb_ctx* ctx, double* ms) {
  SWB_API_BEGIN(ctx);
  if (!ctx->tev0 || !ms) return swb_fail(SWB_EINVAL, "timer not started");
  SWB_CUDA(cudaEventRecord(ctx->tev1, ctx->stream));
  SWB_CUDA(cudaEventSynchronize(ctx->tev1));
  float f = 0.f;
  SWB_CUDA(cudaEventElapsedTime(&f, ctx->tev0, ctx->tev1));
  *ms = f;
  SWB_API_END();
}

int32_t swb_flush_l2(swb_ctx* ctx, int64_t bytes) {
  SWB_API_BEGIN(ctx);
  if (bytes <= 0) bytes = 512LL << 20;
  void* p = swb_scratch(ctx->flush, (size_t)bytes);
  if (!p) return swb_fail(SWB_ECUDA, "cannot allocate the L2 flush buffer");
  SWB_CUDA(cudaMemsetAsync(p, (int)(ctx->launches & 0xff), (size_t)bytes, ctx->stream));
  SWB_CUDA(cudaStreamSynchronize(ctx->stream));
  SWB_API_END();
}

int64_t swb_launch_count(swb_ctx* ctx) { return ctx ? ctx->launches : 0; }

}  // extern "C"
