// ctx.cu -- context, errors, memory helpers of the C ABI (include/lsg.h "core").
#include <cstring>

#include "lsg_common.cuh"

namespace lsg {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

}  // namespace lsg

using namespace lsg;

extern "C" {

int32_t lsg_abi_version(void) { return LSG_ABI_VERSION; }

const char* lsg_last_error(void) { return g_last_error.c_str(); }

lsg_status lsg_device_count(int32_t* n) {
  return guard(__func__, [&] {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *n = c;
  });
}

lsg_status lsg_ctx_create(int32_t device, lsg_ctx* out) {
  return guard(__func__, [&] {
    *out = nullptr;
    int n = 0;
    LSG_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) invalid("lsg_ctx_create: no such device");
    cudaDeviceProp prop{};
    LSG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10 || prop.minor != 0)
      fail(LSG_ECUDA, std::string("lsg: kernels are built for sm_100a; device is ") + prop.name +
                          " (sm_" + std::to_string(prop.major) + std::to_string(prop.minor) + ")");
    auto* c = new lsg_ctx_s();
    c->device = device;
    c->sm_count = prop.multiProcessorCount;
    DeviceGuard g(c);
    LSG_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
    c->stream = c->own;
    c->smem_optin = (int)prop.sharedMemPerBlockOptin;
    c->scratch_get(Ctx::kScratchInit);  // pre-sized: the compute calls do not allocate
    *out = c;
  });
}

lsg_status lsg_ctx_destroy(lsg_ctx ctx) {
  return guard(__func__, [&] {
    if (!ctx) return;
    {
      DeviceGuard g(ctx);
      cudaStreamSynchronize(ctx->stream);
      if (ctx->scratch) cudaFree(ctx->scratch);
      if (ctx->own) cudaStreamDestroy(ctx->own);
    }
    delete ctx;
  });
}

lsg_status lsg_ctx_set_stream(lsg_ctx ctx, void* s) {
  return guard(__func__, [&] { ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own; });
}

lsg_status lsg_ctx_get_stream(lsg_ctx ctx, void** s) {
  return guard(__func__, [&] { *s = ctx->stream; });
}

lsg_status lsg_ctx_sync(lsg_ctx ctx) {
  return guard(__func__, [&] {
    DeviceGuard g(ctx);
    ctx->sync();
  });
}

lsg_status lsg_ctx_launch_count(lsg_ctx ctx, int64_t* n) {
  return guard(__func__, [&] { *n = ctx->launches.load(); });
}

lsg_status lsg_dev_alloc(lsg_ctx ctx, size_t bytes, void** out) {
  return guard(__func__, [&] {
    DeviceGuard g(ctx);
    *out = nullptr;
    LSG_CUDA(cudaMalloc(out, bytes));
  });
}

lsg_status lsg_dev_free(lsg_ctx ctx, void* p) {
  return guard(__func__, [&] {
    DeviceGuard g(ctx);
    LSG_CUDA(cudaFree(p));
  });
}

lsg_status lsg_host_alloc(size_t bytes, void** out) {
  return guard(__func__, [&] {
    *out = nullptr;
    LSG_CUDA(cudaMallocHost(out, bytes));
  });
}

lsg_status lsg_host_free(void* p) {
  return guard(__func__, [&] { LSG_CUDA(cudaFreeHost(p)); });
}

lsg_status lsg_copy(lsg_ctx ctx, void* dst, const void* src, size_t bytes) {
  return guard(__func__, [&] {
    DeviceGuard g(ctx);
    LSG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, ctx->stream));
  });
}

}  // extern "C"
