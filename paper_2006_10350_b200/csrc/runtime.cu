// runtime.cu — context plumbing of libfalkon: errors, workspace arena, launch accounting
// and CUDA-event timing, pointer classification, NCCL (dlopen'ed) communicator.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <mutex>

#include "common.cuh"

namespace falkon {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }
int fail(int code, const std::string &msg) {
  g_last_error = msg;
  return code;
}
const char *last_error_cstr() { return g_last_error.c_str(); }

int ws_get(falkon_ctx *ctx, int slot, size_t bytes, void **out) {
  size_t want = round_up<size_t>(bytes ? bytes : 1, 256) + 256;
  if (ctx->ws_bytes[slot] < want) {
    if (ctx->ws[slot]) {
      FK_CUDA(cudaStreamSynchronize(ctx->stream));
      FK_CUDA(cudaFree(ctx->ws[slot]));
      ctx->ws[slot] = nullptr;
      ctx->ws_bytes[slot] = 0;
    }
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(FALKON_ENOMEM, "workspace allocation of " + std::to_string(want) +
                                     " bytes failed: " + cudaGetErrorString(e));
    }
    FK_CUDA(cudaMemsetAsync(p, 0, want, ctx->stream));
    ctx->ws[slot] = p;
    ctx->ws_bytes[slot] = want;
  }
  *out = ctx->ws[slot];
  return FALKON_OK;
}

LaunchScope::LaunchScope(falkon_ctx *c, int cls_) : ctx(c), cls(cls_) {
  ctx->launches++;
  ctx->t_launches[cls]++;
  if (ctx->opt.kernel_timing) {
    if (!ctx->free_events.empty()) {
      ev = ctx->free_events.back();
      ctx->free_events.pop_back();
    } else {
      cudaEventCreate(&ev.start);
      cudaEventCreate(&ev.stop);
    }
    ev.cls = cls;
    cudaEventRecord(ev.start, ctx->stream);
    timed = true;
  }
}
LaunchScope::~LaunchScope() {
  if (timed) {
    cudaEventRecord(ev.stop, ctx->stream);
    ctx->pending.push_back(ev);
    if (ctx->pending.size() > 4096) resolve_timings(ctx);
  }
}

int resolve_timings(falkon_ctx *ctx) {
  if (ctx->pending.empty()) return FALKON_OK;
  FK_CUDA(cudaStreamSynchronize(ctx->stream));
  for (auto &e : ctx->pending) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, e.start, e.stop) == cudaSuccess) ctx->t_ms[e.cls] += ms;
    ctx->free_events.push_back(e);
  }
  ctx->pending.clear();
  cudaGetLastError();
  return FALKON_OK;
}

bool is_device_ptr(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ------------------------------------------------------------------ NCCL via dlopen
// We only need a handful of entry points; loading NCCL lazily keeps libfalkon free of a
// link-time NCCL dependency and lets it share the libnccl.so.2 torch already loaded.
typedef struct {
  char internal[128];
} nccl_uid_t;
typedef int (*fn_get_uid)(nccl_uid_t *);
typedef int (*fn_init_rank)(void **, int, nccl_uid_t, int);
typedef int (*fn_allreduce)(const void *, void *, size_t, int, int, void *, cudaStream_t);
typedef int (*fn_broadcast)(const void *, void *, size_t, int, int, void *, cudaStream_t);
typedef int (*fn_destroy)(void *);
typedef const char *(*fn_errstr)(int);

static struct {
  std::once_flag once;
  void *h = nullptr;
  fn_get_uid get_uid = nullptr;
  fn_init_rank init_rank = nullptr;
  fn_allreduce allreduce = nullptr;
  fn_broadcast broadcast = nullptr;
  fn_destroy destroy = nullptr;
  fn_errstr errstr = nullptr;
} g_nccl;

// enum values from nccl.h (types only: the functions are resolved with dlsym)
static const int NCCL_INT64 = (int)ncclInt64, NCCL_FLOAT64 = (int)ncclFloat64,
                 NCCL_SUM = (int)ncclSum, NCCL_UINT8 = (int)ncclUint8,
                 NCCL_UINT64 = (int)ncclUint64, NCCL_MIN = (int)ncclMin;

static int nccl_load() {
  std::call_once(g_nccl.once, [] {
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *nm : names) {
      g_nccl.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (g_nccl.h) break;
    }
    if (!g_nccl.h) return;
    g_nccl.get_uid = (fn_get_uid)dlsym(g_nccl.h, "ncclGetUniqueId");
    g_nccl.init_rank = (fn_init_rank)dlsym(g_nccl.h, "ncclCommInitRank");
    g_nccl.allreduce = (fn_allreduce)dlsym(g_nccl.h, "ncclAllReduce");
    g_nccl.broadcast = (fn_broadcast)dlsym(g_nccl.h, "ncclBroadcast");
    g_nccl.destroy = (fn_destroy)dlsym(g_nccl.h, "ncclCommDestroy");
    g_nccl.errstr = (fn_errstr)dlsym(g_nccl.h, "ncclGetErrorString");
  });
  if (!g_nccl.h || !g_nccl.get_uid || !g_nccl.init_rank || !g_nccl.allreduce ||
      !g_nccl.broadcast || !g_nccl.destroy)
    return fail(FALKON_ENCCL, "NCCL (libnccl.so.2) could not be loaded");
  return FALKON_OK;
}

static int nccl_check(int r, const char *what) {
  if (r == 0) return FALKON_OK;
  return fail(FALKON_ENCCL, std::string(what) + " failed: " +
                                (g_nccl.errstr ? g_nccl.errstr(r) : std::to_string(r)));
}

int nccl_get_unique_id(unsigned char id[128]) {
  FK_TRY(nccl_load());
  nccl_uid_t u;
  FK_TRY(nccl_check(g_nccl.get_uid(&u), "ncclGetUniqueId"));
  memcpy(id, u.internal, 128);
  return FALKON_OK;
}

int nccl_comm_init(falkon_ctx *ctx, const unsigned char *id) {
  FK_TRY(nccl_load());
  nccl_uid_t u;
  memcpy(u.internal, id, 128);
  void *comm = nullptr;
  FK_TRY(nccl_check(g_nccl.init_rank(&comm, ctx->world, u, ctx->rank), "ncclCommInitRank"));
  ctx->nccl_comm = comm;
  return FALKON_OK;
}

int nccl_comm_destroy(falkon_ctx *ctx) {
  if (ctx->nccl_comm && g_nccl.destroy) g_nccl.destroy(ctx->nccl_comm);
  ctx->nccl_comm = nullptr;
  return FALKON_OK;
}

int nccl_allreduce_f64(falkon_ctx *ctx, double *buf, int64_t count) {
  if (!ctx->nccl_comm || count == 0) return FALKON_OK;
  LaunchScope ls(ctx, FALKON_T_ALLREDUCE);
  return nccl_check(g_nccl.allreduce(buf, buf, (size_t)count, NCCL_FLOAT64, NCCL_SUM,
                                     ctx->nccl_comm, ctx->stream),
                    "ncclAllReduce");
}

int nccl_allreduce_i64(falkon_ctx *ctx, int64_t *buf, int64_t count) {
  if (!ctx->nccl_comm || count == 0) return FALKON_OK;
  LaunchScope ls(ctx, FALKON_T_ALLREDUCE);
  return nccl_check(g_nccl.allreduce(buf, buf, (size_t)count, NCCL_INT64, NCCL_SUM,
                                     ctx->nccl_comm, ctx->stream),
                    "ncclAllReduce");
}

int nccl_allreduce_min_u64(falkon_ctx *ctx, unsigned long long *buf, int64_t count) {
  if (!ctx->nccl_comm || count == 0) return FALKON_OK;
  LaunchScope ls(ctx, FALKON_T_ALLREDUCE);
  return nccl_check(g_nccl.allreduce(buf, buf, (size_t)count, NCCL_UINT64, NCCL_MIN,
                                     ctx->nccl_comm, ctx->stream),
                    "ncclAllReduce(min)");
}

// In-place broadcast of `bytes` from rank `root` (the distributed preconditioner's panels).
int nccl_broadcast_bytes(falkon_ctx *ctx, void *buf, size_t bytes, int root) {
  if (!ctx->nccl_comm || bytes == 0) return FALKON_OK;
  LaunchScope ls(ctx, FALKON_T_ALLREDUCE);
  return nccl_check(g_nccl.broadcast(buf, buf, bytes, NCCL_UINT8, root, ctx->nccl_comm,
                                     ctx->stream),
                    "ncclBroadcast");
}

}  // namespace falkon
