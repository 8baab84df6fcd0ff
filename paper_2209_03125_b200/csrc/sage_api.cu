// sage_api.cu -- host runtime behind include/sage.h (libsage.so).
//
// Validation, placement choice, occupancy check, launch of the sm_100a
// checksum kernel (sage_kernel.cuh), pinned result readback and host timing
// (the verifier's t0/t1).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <time.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <new>

#include "sage.h"
#include "sage_hash.cuh"
#include "sage_kernel.cuh"

namespace {

thread_local char g_last_error[512] = "";

int fail(int code, const char* fmt, const char* detail = "") {
    snprintf(g_last_error, sizeof(g_last_error), fmt, detail);
    return code;
}

int cuda_fail(cudaError_t e, const char* where) {
    snprintf(g_last_error, sizeof(g_last_error), "%s: %s", where, cudaGetErrorString(e));
    return SAGE_ECUDA;
}

#define CUDA_TRY(expr)                                         \
    do {                                                       \
        cudaError_t _e = (expr);                               \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr);    \
    } while (0)

uint64_t now_ns() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return static_cast<uint64_t>(ts.tv_sec) * 1000000000ull + static_cast<uint64_t>(ts.tv_nsec);
}

constexpr size_t kSmemRegionMax = 64 * 1024;   // 2 CTAs/SM x 64 KiB fits the 228 KB SM
// With the ILP 2 kernel (one CTA per SM) a 128 KiB region still fits in shared memory
// (measured 54.8 ms vs 60.2 ms GLOBAL at 128 KiB).
constexpr size_t kSmemRegionMaxIlp2 = 128 * 1024;
// SAGE_HYBRID: one CTA per SM stages the region's first 192 KiB; larger stages starve
// L1 for the rest (224 KiB: 2x slower), smaller ones stage too little (measured at
// 512 KiB: 128 / 160 / 192 KiB -> 91.4 / 79.0 / 74.1 ms vs 89-94 ms GLOBAL,
// profiles/r01/variants/hybrid_placement*.jsonl).  AUTO uses it for 128 KiB < region
// <= 1 MiB: 61.7 / 75.6 / 18.1 ms (R = 2e4) vs 64.0 / 93.7 / 18.8 ms GLOBAL at
// 256 KiB / 512 KiB / 1 MiB.
constexpr size_t kHybridStage = 192 * 1024, kHybridRegionMax = 1024 * 1024;
// P = 4 (16-B picks) takes SAGE_HYBRID from 256 KiB: 69.5 vs 72.6 ms GLOBAL at
// 256 KiB, 75.9 vs 89.9 ms at the paper's 524,288-B buffer (R = 1e5), 18.3 vs
// 18.9 ms at 1 MiB (R = 2e4); at 128 KiB GLOBAL is faster (65.1 vs 66.3 ms)
// (profiles/r02/c2c48/p4_tiers.jsonl).  P = 8 stays GLOBAL: its staged picks (two
// LDS.128 each) are slower than L1 (117.3 vs 113.8 ms at 512 KiB).
constexpr size_t kHybridRegionMinP4 = 256 * 1024;

using KernelFn = void (*)(const sage::KernelArgs);

// Kernel variant per (P, placement, straddle).  Lowering choices measured on
// B200 with bench/variants.cu: SMEM picks address
// shared memory through an IMAD (ADDR=1) unless chunk addresses straddle a
// 4 GiB boundary; GLOBAL picks use L1-allocating read-only loads.  The round
// loop is unrolled "until it is not possible to unroll further without
// causing instruction cache misses": 32 rounds (a 32 KiB loop body)
// for P=1 from SMEM, 64 is slower; fewer where more unrolling spills.
template <int P> struct Unroll;
template <> struct Unroll<1> { static constexpr int smem = 32, smem_straddle = 16, global = 16; };
template <> struct Unroll<4> { static constexpr int smem = 2, smem_straddle = 2, global = 16; };
// Lowering choices per P (bench/variants.cu; profiles/r01/variants/lowering_scs2_*.jsonl):
//   Addr: pick addressing of non-straddling SMEM regions (ADDR 4 = R6 bracket folded into
//         the chunk-offset IMAD, ADDR 2 = both offsets as IMADs);
//   XsSmem / XsGlobal: 16 = x*M64 as one wide multiply + two chained IMADs.
// P=1 SMEM: ADDR 4 + XS 16 55.33 ms vs 55.93 (ADDR 1, XS 0) at c2a; P=4 SMEM keeps ADDR 2,
// XS 0 (62.1 vs 62.7 ms); GLOBAL: XS 16 is 0.4-1% faster for every P.
template <int P> struct Addr { static constexpr int mode = 1; };
template <> struct Addr<1> { static constexpr int mode = 4; };
template <> struct Addr<4> { static constexpr int mode = 2; };   // measured: 64.52 vs 65.43 ms at 8 KiB
template <int P> struct XsSmem { static constexpr int xs = 0; };
template <> struct XsSmem<1> { static constexpr int xs = 16; };
constexpr int kXsGlobal = 16;
template <> struct Unroll<8> { static constexpr int smem = 1, smem_straddle = 1, global = 1; };

// c2a geometry (P = 1, SMEM, non-straddling, 1024-thread blocks, even block count):
// two logical lane states per hardware thread (ILP 2), one CTA of 1024 threads per SM,
// with PAD registers reserved so the CTA allocates the whole 64 K register file
// (62 registers, allocated per warp in units of 256 = 8 per thread -> 64 x 1024) and
// no other kernel can become resident beside it.  UNROLL and PAD steer
// ptxas' schedule, which moves the attestation time by up to 10%: searches over
// ~700 (UNROLL, PAD, XS, ADDR) schedules (profiles/r01/variants/ilp2_grid*.jsonl,
// schedule_search_429.jsonl; scripts/schedule_search.py)
// found 18 / 7 fastest, 53.76-53.94 vs 54.67-54.87 ms for the previous 16 / 10 on
// three boxes.  It is the fastest implementation of SCS-2 found (DESIGN.md
// section 8): the verifier's margin is the gap to the fastest form (section 11).
constexpr int kIlpSmem = 2, kIlpPad = 7, kIlpUnroll = 18;

uint32_t ilp_for(uint32_t P, bool smem, bool straddle, uint32_t blocks, uint32_t threads) {
    return (P == 1 && smem && !straddle && threads == 1024 && blocks % kIlpSmem == 0) ? kIlpSmem : 1;
}

// SAGE_HYBRID kernels: ILP 2 as above, addressing on the FMA pipe (ADDR 8).  P = 1: 2
// unrolled rounds, 8 reserved registers (64 in all); P = 4: 1 round per trip, no
// reservation (60 registers, allocated as 64).  P = 8 has none (see kHybridRegionMinP4).
constexpr int kHybridUnroll = 2, kHybridPad = 8, kHybridUnrollP4 = 1, kHybridPadP4 = 0;
KernelFn hybrid_kernel(uint32_t P) {
    switch (P) {
        case 1: return sage::sage_checksum_kernel<1, true, false, 16, kHybridUnroll, 8, false, kIlpSmem, kHybridPad>;
        case 4: return sage::sage_checksum_kernel<4, true, false, 16, kHybridUnrollP4, 8, false, kIlpSmem, kHybridPadP4>;
        default: return nullptr;
    }
}

template <int P>
KernelFn kernel_for_p(bool smem, bool straddle, uint32_t ilp) {
    if constexpr (P == 1) {
        if (ilp == kIlpSmem && smem && !straddle)
            return sage::sage_checksum_kernel<1, true, false, XsSmem<1>::xs, kIlpUnroll, Addr<1>::mode, false, kIlpSmem,
                                              kIlpPad>;
    }
    if (smem) {
        return straddle ? sage::sage_checksum_kernel<P, true, true, 0, Unroll<P>::smem_straddle, 0>
                        : sage::sage_checksum_kernel<P, true, false, XsSmem<P>::xs, Unroll<P>::smem, Addr<P>::mode>;
    }
    return sage::sage_checksum_kernel<P, false, true, kXsGlobal, Unroll<P>::global, 0>;
}

KernelFn kernel_for(uint32_t P, bool smem, bool straddle, uint32_t ilp = 1) {
    switch (P) {
        case 1: return kernel_for_p<1>(smem, straddle, ilp);
        case 4: return kernel_for_p<4>(smem, straddle, ilp);
        case 8: return kernel_for_p<8>(smem, straddle, ilp);
        default: return nullptr;
    }
}

// Inclusion-experiment variant (counts reads per chunk); GLOBAL placement.
KernelFn counting_kernel_for(uint32_t P) {
    switch (P) {
        case 1: return sage::sage_checksum_kernel<1, false, true, 0, 1, 0, true>;
        case 4: return sage::sage_checksum_kernel<4, false, true, 0, 1, 0, true>;
        case 8: return sage::sage_checksum_kernel<8, false, true, 0, 1, 0, true>;
        default: return nullptr;
    }
}

}  // namespace

struct sage_ctx {
    int device = 0;
    uint32_t sm_count = 0;
    uint32_t blocks = 0, threads = 0, pick_words = 1, placement = SAGE_AUTO;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    uint64_t* d_raw = nullptr;      // 4 x u64 device result
    uint64_t* h_raw = nullptr;      // 4 x u64 pinned host result
    void* d_stage = nullptr;        // device copy of a host region (sage_attest_host)
    size_t stage_bytes = 0;
    uint64_t launches = 0;
    bool use_tuned = true;          // launch the control-bit-tuned c2a kernel when available
    std::mutex mu;                  // serialises calls that use the ctx-owned buffers
};

namespace {

// Makes the context's device current for the duration of an entry point and
// restores the caller's current device on every return path (a torch user on
// cuda:1 calling into a context on device 0 keeps cuda:1 current).
class DeviceGuard {
  public:
    explicit DeviceGuard(int device) {
        if (cudaGetDevice(&prev_) != cudaSuccess) {
            cudaGetLastError();
            prev_ = -1;
        }
        if (prev_ == device) return;
        const cudaError_t e = cudaSetDevice(device);
        if (e != cudaSuccess) {
            rc_ = cuda_fail(e, "cudaSetDevice");
            return;
        }
        restore_ = prev_ >= 0;
    }
    ~DeviceGuard() {
        if (restore_) cudaSetDevice(prev_);
    }
    int rc() const { return rc_; }
    DeviceGuard(const DeviceGuard&) = delete;
    DeviceGuard& operator=(const DeviceGuard&) = delete;

  private:
    int prev_ = -1;
    bool restore_ = false;
    int rc_ = SAGE_OK;
};

// A buffer the kernel dereferences must be device memory the context's device can
// read: an unregistered host pointer (or another GPU's allocation) would otherwise
// fault inside the kernel and leave the CUDA context unusable.  Managed memory and
// mapped pinned host memory are accepted.
int check_device_ptr(const sage_ctx* c, const void* p, const char* what) {
    if (p == nullptr) return SAGE_OK;
    cudaPointerAttributes at{};
    const cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();                              // not sticky; clear it
        return fail(SAGE_EINVAL, "%s is not a CUDA-visible pointer", what);
    }
    if (at.type == cudaMemoryTypeUnregistered) return fail(SAGE_EINVAL, "%s is host memory, not device memory", what);
    if (at.type == cudaMemoryTypeHost && at.devicePointer == nullptr)
        return fail(SAGE_EINVAL, "%s is pinned host memory without a device mapping", what);
    if (at.type == cudaMemoryTypeDevice && at.device != c->device)
        return fail(SAGE_EINVAL, "%s belongs to another device than the context's", what);
    return SAGE_OK;
}

// Check the SCS-2 preconditions on (bytes, rounds) for P (no pointer involved).
int validate_sizes(const sage_ctx* c, size_t bytes, uint64_t rounds) {
    if (c == nullptr) return fail(SAGE_EINVAL, "null context%s");
    const uint64_t P = c->pick_words;
    if (bytes == 0 || bytes % (4 * P) != 0)
        return fail(SAGE_EINVAL, "region_bytes must be a positive multiple of 4*P%s");
    const uint64_t nc = bytes / (4 * P);
    if ((nc & (nc - 1)) != 0 || nc > (1ull << 32))
        return fail(SAGE_EINVAL, "region chunk count must be a power of two <= 2^32%s");
    if (rounds > 0xFFFFFFFFull) return fail(SAGE_EINVAL, "rounds must be < 2^32%s");
    return SAGE_OK;
}

// Check the SCS-2 preconditions on (region, bytes, rounds) for P.
int validate(const sage_ctx* c, const void* region, size_t bytes, uint64_t rounds) {
    int rc = validate_sizes(c, bytes, rounds);
    if (rc) return rc;
    if (region == nullptr) return fail(SAGE_EINVAL, "null region%s");
    const uint64_t P = c->pick_words;
    const uint64_t align = (4 * P > 16) ? 4 * P : 16;
    if (reinterpret_cast<uintptr_t>(region) % align != 0)
        return fail(SAGE_EINVAL, "region must be 16-byte aligned (32-byte for P=8)%s");
    return check_device_ptr(c, region, "region");
}

// SAGE_AUTO: SMEM when the region fits at 2 CTAs/SM, except P = 8, whose
// random 32-B picks conflict heavily in shared-memory banks and run faster
// from L1 (measured: 1510 vs 1843 cycles per round at 8 KiB).
// The geometry of the ILP 2 kernels: one CTA of 1024 threads per SM (an even block
// count of 1024-thread blocks).  The c2a SMEM kernel is P = 1 only; SAGE_HYBRID has
// P = 1 and P = 4 forms.
bool ilp2_geometry(const sage_ctx* c) { return c->threads == 1024 && c->blocks % kIlpSmem == 0; }
bool hybrid_geometry(const sage_ctx* c) {
    return (c->pick_words == 1 || c->pick_words == 4) && ilp2_geometry(c);
}

size_t smem_region_max(const sage_ctx* c) {
    return c->pick_words == 1 && ilp2_geometry(c) ? kSmemRegionMaxIlp2 : kSmemRegionMax;
}

uint32_t choose_placement(const sage_ctx* c, size_t bytes) {
    if (c->placement != SAGE_AUTO) return c->placement;
    if (c->pick_words == 8) return SAGE_GLOBAL;
    if (bytes <= smem_region_max(c)) return SAGE_SMEM;
    if (bytes <= kHybridRegionMax && hybrid_geometry(c) && (c->pick_words == 1 || bytes >= kHybridRegionMinP4))
        return SAGE_HYBRID;
    return SAGE_GLOBAL;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is only called when a launch
// needs more dynamic shared memory than the kernel already allows on that
// device: setting it on every attestation costs host time between back-to-back
// launches.  Process-wide, guarded by a mutex (contexts may share kernels).
// force = true re-applies the attribute (after a device reset the cache is stale).
int ensure_dyn_smem(int device, const void* fn, int bytes, bool force = false) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, int> set;
    std::lock_guard<std::mutex> lock(mu);
    int& cur = set[{device, fn}];
    if (bytes <= cur && !force) return SAGE_OK;
    CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    cur = bytes;
    return SAGE_OK;
}
int ensure_dyn_smem(int device, KernelFn fn, int bytes, bool force = false) {
    return ensure_dyn_smem(device, reinterpret_cast<const void*>(fn), bytes, force);
}

// The c2a kernel with control-bit-tuned scheduling hints:
// sage_kernel_tuned.cubin next to this library holds the same instructions as the
// embedded c2a kernel with the yield hints of csrc/c2a_yield.json applied (written
// by the build only when the kernel's text is the one the hints were searched
// on).  Loaded once per process; used only if it has the embedded kernel's
// name, registers and static shared memory.  Without the file the embedded
// (untuned) kernel runs.
KernelFn c2a_kernel() {
    return sage::sage_checksum_kernel<1, true, false, XsSmem<1>::xs, kIlpUnroll, Addr<1>::mode, false, kIlpSmem,
                                      kIlpPad>;
}

const void* tuned_c2a() {
    static std::mutex mu;
    static bool tried = false;
    static const void* kernel = nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (tried) return kernel;
    tried = true;
    Dl_info di{};
    if (!dladdr(reinterpret_cast<void*>(&c2a_kernel), &di) || di.dli_fname == nullptr) return nullptr;
    std::string path(di.dli_fname);
    const size_t slash = path.rfind('/');
    path = (slash == std::string::npos ? std::string(".") : path.substr(0, slash)) + "/sage_kernel_tuned.cubin";
    FILE* f = fopen(path.c_str(), "rb");
    if (f == nullptr) return nullptr;
    fclose(f);
    const void* untuned = reinterpret_cast<const void*>(c2a_kernel());
    const char* name = nullptr;
    cudaLibrary_t lib = nullptr;
    cudaKernel_t k = nullptr;
    cudaFuncAttributes a{}, b{};
    if (cudaFuncGetName(&name, untuned) != cudaSuccess ||
        cudaLibraryLoadFromFile(&lib, path.c_str(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
        cudaLibraryGetKernel(&k, lib, name) != cudaSuccess ||
        cudaFuncGetAttributes(&a, untuned) != cudaSuccess ||
        cudaFuncGetAttributes(&b, reinterpret_cast<const void*>(k)) != cudaSuccess ||
        a.numRegs != b.numRegs || a.sharedSizeBytes != b.sharedSizeBytes) {
        cudaGetLastError();                           // not sticky; the embedded kernel runs
        return nullptr;
    }
    kernel = reinterpret_cast<const void*>(k);
    return kernel;
}

// The kernel one attestation of (region, bytes) runs: placement, lane states per
// thread, instantiation and the shared-memory bytes it stages.  region is only used
// for its address (the 4 GiB straddle test), never dereferenced.
struct Plan {
    KernelFn fn = nullptr;
    const void* launch_fn = nullptr;   // what is launched: fn, or its control-bit-tuned copy (c2a)
    uint32_t placement = SAGE_GLOBAL;
    uint32_t ilp = 1;
    size_t dyn = 0;
};

int plan_launch(const sage_ctx* c, const void* region, size_t bytes, bool counting, Plan* out) {
    uint32_t placement = counting ? SAGE_GLOBAL : choose_placement(c, bytes);
    if (placement == SAGE_SMEM && bytes > smem_region_max(c))
        return fail(SAGE_EUNSUPPORTED, "SAGE_SMEM forced but the region exceeds %s",
                    smem_region_max(c) > kSmemRegionMax ? "128 KiB" : "64 KiB");
    const uint64_t lo = reinterpret_cast<uint64_t>(region);
    const bool straddle = (lo >> 32) != ((lo + bytes - 1) >> 32);
    if (placement == SAGE_SMEM && straddle && bytes > kSmemRegionMax) {
        // beyond 64 KiB only the ILP 2 kernel keeps full occupancy, and it needs the
        // 32-bit data pointer of a non-straddling region
        if (c->placement == SAGE_SMEM)
            return fail(SAGE_EUNSUPPORTED, "SAGE_SMEM: a region over 64 KiB must not straddle a 4 GiB boundary%s");
        placement = SAGE_GLOBAL;
    }
    if (placement == SAGE_HYBRID && (!hybrid_geometry(c) || straddle)) {
        if (c->placement == SAGE_HYBRID)
            return fail(SAGE_EUNSUPPORTED, "SAGE_HYBRID needs P=1 or 4, 1024-thread blocks, an even block count and a "
                                           "region inside one 4 GiB window%s");
        placement = SAGE_GLOBAL;                    // AUTO: a straddling region runs GLOBAL
    }
    const bool hybrid = placement == SAGE_HYBRID;
    const bool smem = placement == SAGE_SMEM;
    uint32_t ilp = counting ? 1 : ilp_for(c->pick_words, smem, straddle, c->blocks, c->threads);
    KernelFn fn = counting ? counting_kernel_for(c->pick_words) : kernel_for(c->pick_words, smem, straddle, ilp);
    if (hybrid) {
        ilp = kIlpSmem;
        fn = hybrid_kernel(c->pick_words);
    }
    if (fn == nullptr) return fail(SAGE_EINVAL, "pick_words must be 1, 4 or 8%s");
    out->fn = fn;
    out->launch_fn = reinterpret_cast<const void*>(fn);
    if (fn == c2a_kernel() && c->use_tuned) {
        const void* t = tuned_c2a();
        if (t) out->launch_fn = t;
    }
    out->placement = placement;
    out->ilp = ilp;
    out->dyn = smem ? bytes : hybrid ? (bytes < kHybridStage ? bytes : kHybridStage) : 0;
    return SAGE_OK;
}

int launch(sage_ctx* c, uint64_t nonce, const void* region, size_t bytes, uint64_t rounds, uint64_t* raw,
           uint64_t* per_warp, uint32_t* placement_used, uint32_t* counts = nullptr, uint32_t* ilp_used = nullptr,
           uint32_t* tuned_used = nullptr) {
    Plan plan;
    int prc = plan_launch(c, region, bytes, counts != nullptr, &plan);
    if (prc) return prc;
    const void* fn = plan.launch_fn;
    const uint32_t placement = plan.placement, ilp = plan.ilp;
    const size_t dyn = plan.dyn;
    if (dyn) {
        int rc = ensure_dyn_smem(c->device, fn, static_cast<int>(dyn));
        if (rc) return rc;
    }
    sage::KernelArgs args{};
    args.region = static_cast<const uint32_t*>(region);
    args.nonce = nonce;
    args.nc_mask = static_cast<uint32_t>(bytes / (4ull * c->pick_words) - 1);
    args.rounds = static_cast<uint32_t>(rounds);
    args.region_bytes = static_cast<uint32_t>(dyn);   // bytes staged in shared memory
    args.raw = raw;
    args.per_warp = per_warp;
    args.counts = counts;
    sage::fill_tables(args, c->pick_words);
#ifdef SAGE_BOUNDS_CHECK
    // bounds-checked build only: a negative control for the checks -- tell the kernel
    // one chunk less is staged than its picks can reach, which must trap
    if (dyn && getenv("SAGE_CHECK_SELFTEST")) args.region_bytes -= 4u * c->pick_words;
#endif
    void* params[] = {&args};
    cudaError_t le = cudaLaunchKernel(fn, dim3(c->blocks / ilp), dim3(c->threads), params, dyn, c->stream);
    if (le == cudaErrorInvalidValue && dyn) {
        // the cached shared-memory limit is stale (e.g. cudaDeviceReset): re-apply it once
        cudaGetLastError();
        int rc = ensure_dyn_smem(c->device, fn, static_cast<int>(dyn), true);
        if (rc) return rc;
        le = cudaLaunchKernel(fn, dim3(c->blocks / ilp), dim3(c->threads), params, dyn, c->stream);
    }
    if (le != cudaSuccess) {
        cudaGetLastError();
        return cuda_fail(le, "checksum kernel launch");
    }
    c->launches++;
    if (placement_used) *placement_used = placement;
    if (ilp_used) *ilp_used = ilp;
    if (tuned_used) *tuned_used = fn != reinterpret_cast<const void*>(plan.fn);
    return SAGE_OK;
}

void fill_result(const sage_ctx* c, const uint64_t raw[4], uint64_t t0, uint64_t t1, uint64_t va, uint32_t placement,
                 uint32_t ilp, uint32_t tuned, sage_result* out) {
    sage_decode_raw(raw, out);
    out->ilp = ilp;
    out->tuned = tuned;
    out->elapsed_ns = t1 - t0;
    out->region_va = va;
    out->placement = placement;
    out->blocks = c->blocks;
    out->threads = c->threads;
    out->pick_words = c->pick_words;
}

// attest synchronously over a device region already validated (device already current)
int attest_device(sage_ctx* c, uint64_t nonce, const void* region, size_t bytes, uint64_t rounds,
                  uint64_t* per_warp, sage_result* out, const void* host_src, uint32_t* counts = nullptr) {
    const uint64_t t0 = now_ns();
    if (host_src) CUDA_TRY(cudaMemcpyAsync(const_cast<void*>(region), host_src, bytes, cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(cudaMemsetAsync(c->d_raw, 0, 4 * sizeof(uint64_t), c->stream));
    uint32_t placement = 0, ilp = 1, tuned = 0;
    int rc = launch(c, nonce, region, bytes, rounds, c->d_raw, per_warp, &placement, counts, &ilp, &tuned);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(c->h_raw, c->d_raw, 4 * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    const uint64_t t1 = now_ns();
    fill_result(c, c->h_raw, t0, t1, reinterpret_cast<uint64_t>(region), placement, ilp, tuned, out);
    return SAGE_OK;
}

int ensure_stage(sage_ctx* c, size_t bytes) {
    if (c->stage_bytes >= bytes) return SAGE_OK;
    if (c->d_stage) cudaFree(c->d_stage);
    c->d_stage = nullptr;
    c->stage_bytes = 0;
    cudaError_t e = cudaMalloc(&c->d_stage, bytes);
    if (e != cudaSuccess) return fail(SAGE_ENOMEM, "cudaMalloc of the host-region staging buffer failed%s");
    c->stage_bytes = bytes;
    return SAGE_OK;
}

// Dynamic shared-memory limits of the kernels this context can stage into, set
// once when the context is created so that later calls (sage_query, launches)
// do not change kernel attributes.
int prepare_kernels(const sage_ctx* c) {
    const uint32_t ilp = ilp_for(c->pick_words, true, false, c->blocks, c->threads);
    int rc = ensure_dyn_smem(c->device, kernel_for(c->pick_words, true, false, ilp),
                             static_cast<int>(smem_region_max(c)));
    if (rc == SAGE_OK) rc = ensure_dyn_smem(c->device, kernel_for(c->pick_words, true, true), static_cast<int>(kSmemRegionMax));
    if (rc == SAGE_OK && hybrid_geometry(c))
        rc = ensure_dyn_smem(c->device, hybrid_kernel(c->pick_words), static_cast<int>(kHybridStage));
    if (rc == SAGE_OK && c->use_tuned && kernel_for(c->pick_words, true, false, ilp) == c2a_kernel()) {
        const void* t = tuned_c2a();
        if (t) rc = ensure_dyn_smem(c->device, t, static_cast<int>(smem_region_max(c)));
    }
    return rc;
}

}  // namespace

extern "C" {

int sage_checksum_init(const sage_config* cfg, sage_ctx** out) {
    if (out == nullptr) return fail(SAGE_EINVAL, "out is null%s");
    sage_config d{};
    if (cfg) d = *cfg;
    if (d.threads == 0) d.threads = 1024;
    if (d.pick_words == 0) d.pick_words = 1;
    if (d.threads % 32 != 0 || d.threads > 1024) return fail(SAGE_EINVAL, "threads must be a multiple of 32, <= 1024%s");
    if (d.pick_words != 1 && d.pick_words != 4 && d.pick_words != 8)
        return fail(SAGE_EINVAL, "pick_words must be 1, 4 or 8%s");
    if (d.placement > SAGE_HYBRID) return fail(SAGE_EINVAL, "unknown placement%s");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (d.device < 0 || d.device >= ndev) return fail(SAGE_EINVAL, "device ordinal out of range%s");
    DeviceGuard dg(d.device);
    if (dg.rc()) return dg.rc();
    int sms = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d.device));

    sage_ctx* c = new (std::nothrow) sage_ctx();
    if (!c) return fail(SAGE_ENOMEM, "context allocation failed%s");
    c->device = d.device;
    c->sm_count = static_cast<uint32_t>(sms);
    c->threads = d.threads;
    c->blocks = d.blocks ? d.blocks : 2u * static_cast<uint32_t>(sms);
    c->pick_words = d.pick_words;
    c->placement = d.placement;
    c->use_tuned = getenv("SAGE_NO_TUNED") == nullptr;      // A/B switch
    cudaError_t e;
    if (d.stream) {
        c->stream = static_cast<cudaStream_t>(d.stream);
    } else {
        // a blocking stream: its work is ordered with the legacy default stream (the one
        // torch and plain CUDA code use unless told otherwise), so buffers written there
        // before an attestation call are complete when the kernel reads them
        e = cudaStreamCreateWithFlags(&c->stream, cudaStreamDefault);
        if (e != cudaSuccess) { delete c; return cuda_fail(e, "cudaStreamCreate"); }
        c->own_stream = true;
    }
    e = cudaMalloc(&c->d_raw, 4 * sizeof(uint64_t));
    if (e != cudaSuccess) { sage_checksum_destroy(c); return fail(SAGE_ENOMEM, "cudaMalloc result%s"); }
    e = cudaMallocHost(&c->h_raw, 4 * sizeof(uint64_t));
    if (e != cudaSuccess) { sage_checksum_destroy(c); return fail(SAGE_ENOMEM, "cudaMallocHost result%s"); }
    const int rc = prepare_kernels(c);
    if (rc) { sage_checksum_destroy(c); return rc; }
    *out = c;
    return SAGE_OK;
}

int sage_attest(sage_ctx* ctx, uint64_t nonce, const void* region, size_t region_bytes, uint64_t rounds,
                sage_result* out) {
    return sage_attest_debug(ctx, nonce, region, region_bytes, rounds, nullptr, out);
}

int sage_attest_debug(sage_ctx* ctx, uint64_t nonce, const void* region, size_t region_bytes, uint64_t rounds,
                      uint64_t* per_warp_out, sage_result* out) {
    int rc = validate(ctx, region, region_bytes, rounds);
    if (rc) return rc;
    if (out == nullptr) return fail(SAGE_EINVAL, "out is null%s");
    rc = check_device_ptr(ctx, per_warp_out, "per_warp_out");
    if (rc) return rc;
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceGuard dg(ctx->device);
    if (dg.rc()) return dg.rc();
    sage_result tmp;
    rc = attest_device(ctx, nonce, region, region_bytes, rounds, per_warp_out, &tmp, nullptr);
    if (rc) return rc;
    *out = tmp;
    return SAGE_OK;
}

int sage_attest_async(sage_ctx* ctx, uint64_t nonce, const void* region, size_t region_bytes, uint64_t rounds,
                      uint64_t* raw_out, uint64_t* per_warp_out) {
    int rc = validate(ctx, region, region_bytes, rounds);
    if (rc) return rc;
    if (raw_out == nullptr) return fail(SAGE_EINVAL, "raw_out is null%s");
    if ((rc = check_device_ptr(ctx, raw_out, "raw_out")) || (rc = check_device_ptr(ctx, per_warp_out, "per_warp_out")))
        return rc;
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceGuard dg(ctx->device);
    if (dg.rc()) return dg.rc();
    return launch(ctx, nonce, region, region_bytes, rounds, raw_out, per_warp_out, nullptr);
}

int sage_attest_coverage(sage_ctx* ctx, uint64_t nonce, const void* region, size_t region_bytes, uint64_t rounds,
                         uint32_t* counts_out, sage_result* out) {
    int rc = validate(ctx, region, region_bytes, rounds);
    if (rc) return rc;
    if (counts_out == nullptr || out == nullptr) return fail(SAGE_EINVAL, "null pointer%s");
    rc = check_device_ptr(ctx, counts_out, "counts_out");
    if (rc) return rc;
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceGuard dg(ctx->device);
    if (dg.rc()) return dg.rc();
    CUDA_TRY(cudaMemsetAsync(counts_out, 0, region_bytes / (4ull * ctx->pick_words) * sizeof(uint32_t), ctx->stream));
    sage_result tmp;
    rc = attest_device(ctx, nonce, region, region_bytes, rounds, nullptr, &tmp, nullptr, counts_out);
    if (rc) return rc;
    *out = tmp;
    return SAGE_OK;
}

int sage_kernel_hash(sage_ctx* ctx, const uint8_t* r, size_t r_len, const void* code, size_t code_len,
                     uint8_t* h_out, uint64_t* elapsed_ns) {
    if (ctx == nullptr || h_out == nullptr || (r == nullptr && r_len) || (code == nullptr && code_len))
        return fail(SAGE_EINVAL, "null pointer%s");
    if (r_len > static_cast<size_t>(sage::kHashRMax)) return fail(SAGE_EINVAL, "r longer than %s bytes", "128");
    if (code_len) {
        const int rc = check_device_ptr(ctx, code, "code");
        if (rc) return rc;
    }
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceGuard dg(ctx->device);
    if (dg.rc()) return dg.rc();
    sage::HashArgs args{};
    args.code = static_cast<const uint8_t*>(code);
    args.code_len = code_len;
    args.out = reinterpret_cast<uint8_t*>(ctx->d_raw);
    args.r_len = static_cast<uint32_t>(r_len);
    if (r_len) memcpy(args.r, r, r_len);
    const uint64_t t0 = now_ns();
    sage::sage_sha256_kernel<<<1, 64, 0, ctx->stream>>>(args);
    CUDA_TRY(cudaGetLastError());
    ctx->launches++;
    CUDA_TRY(cudaMemcpyAsync(ctx->h_raw, ctx->d_raw, 32, cudaMemcpyDeviceToHost, ctx->stream));
    CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    const uint64_t t1 = now_ns();
    memcpy(h_out, ctx->h_raw, 32);
    if (elapsed_ns) *elapsed_ns = t1 - t0;
    return SAGE_OK;
}

int sage_decode_raw(const uint64_t raw[4], sage_result* out) {
    if (raw == nullptr || out == nullptr) return fail(SAGE_EINVAL, "null pointer%s");
    memset(out, 0, sizeof(*out));
    out->checksum = raw[0];
    out->cycles = raw[1];
    const uint64_t start = ~raw[2];
    out->device_ns = raw[3] >= start ? raw[3] - start : 0;
    return SAGE_OK;
}

int sage_attest_host(sage_ctx* ctx, uint64_t nonce, const void* host_region, size_t region_bytes, uint64_t rounds,
                     sage_result* out) {
    if (ctx == nullptr || host_region == nullptr || out == nullptr) return fail(SAGE_EINVAL, "null pointer%s");
    // sizes first: an invalid call must not reallocate the staging buffer (its VA is
    // what a verifier precomputed the expected checksum for, sage_host_region_va)
    int rc = validate_sizes(ctx, region_bytes, rounds);
    if (rc) return rc;
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceGuard dg(ctx->device);
    if (dg.rc()) return dg.rc();
    rc = ensure_stage(ctx, region_bytes);
    if (rc) return rc;
    rc = validate(ctx, ctx->d_stage, region_bytes, rounds);
    if (rc) return rc;
    sage_result tmp;
    rc = attest_device(ctx, nonce, ctx->d_stage, region_bytes, rounds, nullptr, &tmp, host_region);
    if (rc) return rc;
    *out = tmp;
    return SAGE_OK;
}

int sage_host_region_va(sage_ctx* ctx, size_t region_bytes, uint64_t* va_out) {
    if (ctx == nullptr || va_out == nullptr) return fail(SAGE_EINVAL, "null pointer%s");
    int rc = validate_sizes(ctx, region_bytes, 0);
    if (rc) return rc;
    std::lock_guard<std::mutex> lock(ctx->mu);
    DeviceGuard dg(ctx->device);
    if (dg.rc()) return dg.rc();
    rc = ensure_stage(ctx, region_bytes);
    if (rc) return rc;
    *va_out = reinterpret_cast<uint64_t>(ctx->d_stage);
    return SAGE_OK;
}

int sage_placement_for(sage_ctx* ctx, size_t region_bytes, uint32_t* placement_out) {
    if (ctx == nullptr || placement_out == nullptr) return fail(SAGE_EINVAL, "null pointer%s");
    *placement_out = choose_placement(ctx, region_bytes);
    return SAGE_OK;
}

int sage_kernel_symbol(sage_ctx* ctx, uint64_t region_va, size_t region_bytes, char* buf, size_t buf_len) {
    if (ctx == nullptr || buf == nullptr || buf_len == 0) return fail(SAGE_EINVAL, "null pointer%s");
    int rc = validate_sizes(ctx, region_bytes, 0);
    if (rc) return rc;
    Plan plan;
    rc = plan_launch(ctx, reinterpret_cast<const void*>(region_va), region_bytes, false, &plan);
    if (rc) return rc;
    DeviceGuard dg(ctx->device);
    if (dg.rc()) return dg.rc();
    const char* name = nullptr;
    CUDA_TRY(cudaFuncGetName(&name, reinterpret_cast<const void*>(plan.fn)));
    const size_t n = strlen(name);
    if (n + 1 > buf_len) return fail(SAGE_EINVAL, "buffer too small for the kernel symbol%s");
    memcpy(buf, name, n + 1);
    return SAGE_OK;
}

int sage_device_uuid(sage_ctx* ctx, uint8_t uuid_out[16]) {
    if (ctx == nullptr || uuid_out == nullptr) return fail(SAGE_EINVAL, "null pointer%s");
    cudaDeviceProp prop{};
    CUDA_TRY(cudaGetDeviceProperties(&prop, ctx->device));
    memcpy(uuid_out, prop.uuid.bytes, 16);
    return SAGE_OK;
}

int sage_query(sage_ctx* ctx, sage_info* out) {
    if (ctx == nullptr || out == nullptr) return fail(SAGE_EINVAL, "null pointer%s");
    DeviceGuard dg(ctx->device);
    if (dg.rc()) return dg.rc();
    sage_info info{};
    info.device = ctx->device;
    info.sm_count = ctx->sm_count;
    info.blocks = ctx->blocks;
    info.threads = ctx->threads;
    info.pick_words = ctx->pick_words;
    info.placement = ctx->placement;
    info.smem_region_max = smem_region_max(ctx);
    const uint32_t ilp = ilp_for(ctx->pick_words, true, false, ctx->blocks, ctx->threads);
    info.ilp_smem = ilp;
    // read-only: the dynamic shared-memory limit of the SMEM kernel was set at init
    KernelFn fs = kernel_for(ctx->pick_words, true, false, ilp), fg = kernel_for(ctx->pick_words, false, true);
    int occ = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fs, static_cast<int>(ctx->threads), kSmemRegionMax));
    info.ctas_per_sm_smem = static_cast<uint32_t>(occ);
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fg, static_cast<int>(ctx->threads), 0));
    info.ctas_per_sm_global = static_cast<uint32_t>(occ);
    cudaFuncAttributes fa;
    CUDA_TRY(cudaFuncGetAttributes(&fa, fs));
    info.regs_per_thread = static_cast<uint32_t>(fa.numRegs);
    *out = info;
    return SAGE_OK;
}

uint64_t sage_launch_count(const sage_ctx* ctx) { return ctx ? ctx->launches : 0; }

void* sage_stream(const sage_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

void sage_checksum_destroy(sage_ctx* ctx) {
    if (!ctx) return;
    DeviceGuard dg(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->d_raw) cudaFree(ctx->d_raw);
    if (ctx->h_raw) cudaFreeHost(ctx->h_raw);
    if (ctx->d_stage) cudaFree(ctx->d_stage);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char* sage_strerror(int code) {
    switch (code) {
        case SAGE_OK: return "ok";
        case SAGE_EINVAL: return "invalid argument";
        case SAGE_EUNSUPPORTED: return "unsupported configuration";
        case SAGE_ENOMEM: return "out of memory";
        case SAGE_ECUDA: return "CUDA error";
        default: return "unknown error";
    }
}

const char* sage_last_error(void) { return g_last_error; }

}  // extern "C"
