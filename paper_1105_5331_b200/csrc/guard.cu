// Guard bands around every device allocation (built into every library; active only in the
// -DCPFIT_GUARD variant, where common.cuh routes cudaMalloc / cudaFree here). Each allocation is
// [4 KB guard | user bytes | 4 KB guard], guards filled with 0xA5; a free, or
// cpfit_debug_guard_check(), reads the guards back and counts any changed byte as an
// out-of-bounds write by a kernel (or copy) of this library.
#define CPFIT_GUARD_IMPL
#include "../../include/cpfit_gpu.h"
#include "common.cuh"

#include <cstdio>
#include <map>
#include <mutex>
#include <vector>

namespace cpfit_gpu {
namespace {
constexpr size_t kGuard = 4096;
constexpr unsigned char kPat = 0xA5;
struct Alloc {
    char* base;
    size_t bytes;
};
std::mutex& mu() {
    static std::mutex* m = new std::mutex();
    return *m;
}
std::map<void*, Alloc>& live() {
    static auto* m = new std::map<void*, Alloc>();
    return *m;
}
long long g_violations = 0;

long long check_one(void* user, const Alloc& a) {
    std::vector<unsigned char> h(2 * kGuard);
    if (cudaMemcpy(h.data(), a.base, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(h.data() + kGuard, a.base + kGuard + a.bytes, kGuard, cudaMemcpyDeviceToHost) != cudaSuccess)
        return 0;
    long long bad = 0;
    for (size_t i = 0; i < h.size(); ++i) bad += h[i] != kPat;
    if (bad)
        std::fprintf(stderr, "cpfit guard: %lld corrupted guard bytes around %p (%zu bytes)\n", bad, user, a.bytes);
    return bad ? 1 : 0;
}
}  // namespace

cudaError_t guard_malloc(void** p, size_t bytes) {
    char* base = nullptr;
    cudaError_t e = cudaMalloc(&base, bytes + 2 * kGuard);
    if (e != cudaSuccess) return e;
    cudaMemset(base, kPat, kGuard);
    cudaMemset(base + kGuard + bytes, kPat, kGuard);
    *p = base + kGuard;
    std::lock_guard<std::mutex> lk(mu());
    live()[*p] = Alloc{base, bytes};
    return cudaSuccess;
}

cudaError_t guard_free(void* p) {
    if (!p) return cudaSuccess;
    Alloc a{};
    {
        std::lock_guard<std::mutex> lk(mu());
        auto it = live().find(p);
        if (it == live().end()) return cudaFree(p);
        a = it->second;
        live().erase(it);
    }
    cudaDeviceSynchronize();
    const long long v = check_one(p, a);
    {
        std::lock_guard<std::mutex> lk(mu());
        g_violations += v;
    }
    return cudaFree(a.base);
}
}  // namespace cpfit_gpu

extern "C" int cpfit_debug_guard_check(int64_t* violations, int64_t* live_allocations) {
#ifdef CPFIT_GUARD
    using namespace cpfit_gpu;
    cudaDeviceSynchronize();
    std::lock_guard<std::mutex> lk(mu());
    long long v = 0;
    for (auto& kv : live()) v += check_one(kv.first, kv.second);
    g_violations += v;
    if (violations) *violations = g_violations;
    if (live_allocations) *live_allocations = (int64_t)live().size();
    return 0;
#else
    if (violations) *violations = -1;  // not a guard build
    if (live_allocations) *live_allocations = 0;
    return 0;
#endif
}
