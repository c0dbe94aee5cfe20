// comm.cu — the library's NCCL communicator (SURVEY §8(b) multi-GPU contract, §8(e)).
//
// libcpi does not link NCCL: it is loaded at run time (dlopen of libnccl.so.2) the first time a
// context with world > 1 is created, so single-GPU users and the CPU tier never need it.  A process
// that already holds an NCCL (e.g. torch's) gets that same library back (dlopen by soname).
// Also the two tiny elementwise kernels the plane all-reduce needs (fp32 <-> fp64).
#include <dlfcn.h>

#include <mutex>

#include "kernels.h"

namespace cpi {

namespace {
NcclApi g_api{};
bool g_ok = false;
std::once_flag g_once;

template <class F>
bool sym(void* h, const char* name, F& f) {
    f = reinterpret_cast<F>(dlsym(h, name));
    return f != nullptr;
}
}  // namespace

const NcclApi* nccl_api() {
    std::call_once(g_once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
        if (!h) return;
        g_ok = sym(h, "ncclGetUniqueId", g_api.get_unique_id) && sym(h, "ncclCommInitRank", g_api.comm_init_rank) &&
               sym(h, "ncclCommDestroy", g_api.comm_destroy) && sym(h, "ncclAllReduce", g_api.all_reduce) &&
               sym(h, "ncclReduceScatter", g_api.reduce_scatter) && sym(h, "ncclAllGather", g_api.all_gather) &&
               sym(h, "ncclGroupStart", g_api.group_start) &&
               sym(h, "ncclGroupEnd", g_api.group_end) && sym(h, "ncclGetErrorString", g_api.error_string);
    });
    return g_ok ? &g_api : nullptr;
}

namespace {
__global__ void f32_to_f64_kernel(const float* __restrict__ a, double* __restrict__ b, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        b[i] = static_cast<double>(a[i]);
}
__global__ void f64_to_f32_kernel(const double* __restrict__ a, float* __restrict__ b, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        b[i] = static_cast<float>(a[i]);
}
}  // namespace

cudaError_t launch_f32_to_f64(const float* a, double* b, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int64_t blocks = (n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096;
    f32_to_f64_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(a, b, n);
    return cudaGetLastError();
}
cudaError_t launch_f64_to_f32(const double* a, float* b, int64_t n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    const int64_t blocks = (n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096;
    f64_to_f32_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(a, b, n);
    return cudaGetLastError();
}

}  // namespace cpi
