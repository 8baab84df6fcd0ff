// adversary_lib.cu -- test-only C ABI over timing-adversary kernels (libsage_adv.so).
//
// NOT PART OF THE PRODUCT.  SAGE's security argument is that a modified
// verification function is either wrong or measurably slower (Table 1
// Exp 1 vs Exp 2).  This library exposes adversary
// versions of the product's c2a kernel -- the lab template (bench/sage_lab.cuh,
// whose main loop with every knob off equals the product's, tests/test_sass_evidence.py)
// with result-neutral instructions injected, re-scheduled by an attacker's own
// schedule search (scripts/schedule_search.py --extra), or reading a relocated
// clean copy of the region (memory-copy attack) -- so that tests/test_gpu_adversary.py
// can interleave them with the product's sage_attest and apply the verifier.
// Each call does what sage_attest does around the kernel (32-B memset, launch,
// 32-B D2H into pinned memory, stream sync) and times it the same way (host
// CLOCK_MONOTONIC, the verifier's t1 - t0).
#include <cuda_runtime.h>
#include <time.h>

#include <cstdint>
#include <cstring>
#include <mutex>

#include "sage_lab.cuh"

namespace {

using Fn = void (*)(const sage_lab::KernelArgs);
struct Adv {
    const char* name;
    Fn fn;
    int ilp;
    int memcopy;       // reads a copy at region + copy_delta while folding region's address
    int stage = -1;    // shared-memory bytes staged: -1 = the whole region (SMEM), 0 = none
                       // (GLOBAL), > 0 = a prefix of that many bytes (HYBRID)
    int probe = 0;     // 1: a side experiment, not part of the adversary test
};

// <P, SMEM, STRADDLE, XS, UNROLL, ADDR, LD, EXTRA, COUNT, EVERY, ILP, PROBE, PAD, SYNC, FEXTRA, MEMCOPY>
// The product's c2a kernel is <1, SMEM, nostraddle, XS 16, UNROLL 18, ADDR 4, ILP 2, PAD 7>.
// The attacker's schedules: the fastest points of scripts/schedule_search.py run over
// the adversary's own kernel (UNROLL 8-36 x PAD 0-12 for +1 IMAD / round, 377 points;
// UNROLL 7..35 step 7 x PAD 0-12 for +1 IMAD / 7 rounds, 65 points; profiles/r02/):
// UNROLL 9 / PAD 1 (+0.054% vs the product) and UNROLL 7 / PAD 10 (+1.27%).
#ifndef ADV_ATK_U
#define ADV_ATK_U 9
#define ADV_ATK_PAD 1
#endif
#ifndef ADV_ATK7_U
#define ADV_ATK7_U 7
#define ADV_ATK7_PAD 10
#endif
const Adv kAdv[] = {
    {"+1 IMAD / round (product schedule)",
     sage_lab::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, -1, false, 1, 2, 0, 7>, 2, 0},
    {"+1 ALU op / 18 rounds (product schedule)",
     sage_lab::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, 1, false, 18, 2, 0, 7>, 2, 0},
    {"+1 IMAD / round (attacker-searched schedule, 2nd best: UNROLL 17 / PAD 7)",
     sage_lab::sage_checksum_kernel<1, true, false, 16, 17, 4, 0, -1, false, 1, 2, 0, 7>, 2, 0},
    {"+1 IMAD / round (attacker-searched schedule)",
     sage_lab::sage_checksum_kernel<1, true, false, 16, ADV_ATK_U, 4, 0, -1, false, 1, 2, 0, ADV_ATK_PAD>, 2, 0},
    {"+1 IMAD / 7 rounds (attacker-searched schedule)",
     sage_lab::sage_checksum_kernel<1, true, false, 16, ADV_ATK7_U, 4, 0, -1, false, 7, 2, 0, ADV_ATK7_PAD>, 2, 0},
    {"memory copy: stage a clean copy, fold the original address",
     sage_lab::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, 0, false, 0, 2, 0, 7, 0, 0, 1>, 2, 1},
    // side experiments (scripts/memcopy_probe.py): the memory-copy attack on the other
    // placements -- GLOBAL (the product's P=1 GLOBAL kernel reading dp + delta) and
    // SAGE_HYBRID (staged prefix and in-place part both from the copy)
    {"memory copy on GLOBAL placement",
     sage_lab::sage_checksum_kernel<1, false, true, 16, 16, 0, 0, 0, false, 0, 1, 0, 0, 0, 0, 1>, 1, 1, 0, 1},
    {"memory copy on SAGE_HYBRID placement",
     sage_lab::sage_checksum_kernel<1, true, false, 16, 2, 8, 0, 0, false, 0, 2, 0, 8, 0, 0, 1>, 2, 1, 196608, 1},
};
constexpr int kCount = sizeof(kAdv) / sizeof(kAdv[0]);

struct State {
    bool ready = false;
    int device = -1, sms = 0;
    cudaStream_t stream = nullptr;
    uint64_t* d_raw = nullptr;
    uint64_t* h_raw = nullptr;
    std::mutex mu;
} g;

uint64_t now_ns() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return uint64_t(ts.tv_sec) * 1000000000ull + uint64_t(ts.tv_nsec);
}

int ensure(int device) {
    if (g.ready && g.device == device) return 0;
    if (cudaSetDevice(device) != cudaSuccess) return -4;
    if (cudaDeviceGetAttribute(&g.sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -4;
    if (cudaStreamCreateWithFlags(&g.stream, cudaStreamDefault) != cudaSuccess) return -4;
    if (cudaMalloc(&g.d_raw, 32) != cudaSuccess || cudaMallocHost(&g.h_raw, 32) != cudaSuccess) return -3;
    for (const Adv& a : kAdv)
        if (a.stage != 0 && cudaFuncSetAttribute(reinterpret_cast<const void*>(a.fn),
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 a.stage > 0 ? a.stage : 65536) != cudaSuccess)
            return -4;
    g.device = device;
    g.ready = true;
    return 0;
}

}  // namespace

extern "C" {

int adv_count(void) { return kCount; }

const char* adv_name(int k) { return (k >= 0 && k < kCount) ? kAdv[k].name : nullptr; }

int adv_memcopy(int k) { return (k >= 0 && k < kCount) ? kAdv[k].memcopy : -1; }

int adv_probe(int k) { return (k >= 0 && k < kCount) ? kAdv[k].probe : -1; }

/* One attestation with adversary k at full occupancy (2 x SMs x 1024 logical
 * threads, P = 1; region_bytes a power of two >= 16, <= 64 KiB for kernels that
 * stage the whole region).  copy_delta: for memory-copy adversaries, the byte offset of the clean
 * copy the kernel really reads (region + copy_delta); the folded address stays
 * `region`.  per_warp (device, may be NULL) gets the warp partials.  Returns 0, or
 * -1 bad argument, -3 allocation, -4 CUDA error. */
int adv_attest(int k, int device, uint64_t nonce, const void* region, size_t region_bytes, uint32_t rounds,
               int64_t copy_delta, uint64_t* per_warp, uint64_t* checksum, uint64_t* elapsed_ns) {
    if (k < 0 || k >= kCount || region == nullptr || checksum == nullptr || elapsed_ns == nullptr) return -1;
    if (region_bytes < 16 || (region_bytes & (region_bytes - 1))) return -1;
    if (kAdv[k].stage < 0 && region_bytes > 65536) return -1;
    const size_t dyn = kAdv[k].stage < 0 ? region_bytes
                       : (kAdv[k].stage > 0 && region_bytes > size_t(kAdv[k].stage) ? size_t(kAdv[k].stage) : 0);
    if (kAdv[k].stage > 0 && dyn == 0) return -1;      // HYBRID needs a region above its stage
    std::lock_guard<std::mutex> lock(g.mu);
    int rc = ensure(device);
    if (rc) return rc;
    sage_lab::KernelArgs a{};
    a.region = static_cast<const uint32_t*>(region);
    a.nonce = nonce;
    a.nc_mask = static_cast<uint32_t>(region_bytes / 4 - 1);
    a.rounds = rounds;
    a.region_bytes = static_cast<uint32_t>(dyn);
    a.raw = g.d_raw;
    a.per_warp = per_warp;
    a.copy_delta = copy_delta;
    sage_lab::fill_tables(a, 1);
    const int grid = 2 * g.sms / kAdv[k].ilp;
    const uint64_t t0 = now_ns();
    if (cudaMemsetAsync(g.d_raw, 0, 32, g.stream) != cudaSuccess) return -4;
    kAdv[k].fn<<<grid, 1024, dyn, g.stream>>>(a);
    if (cudaGetLastError() != cudaSuccess) return -4;
    if (cudaMemcpyAsync(g.h_raw, g.d_raw, 32, cudaMemcpyDeviceToHost, g.stream) != cudaSuccess) return -4;
    if (cudaStreamSynchronize(g.stream) != cudaSuccess) return -4;
    const uint64_t t1 = now_ns();
    *checksum = g.h_raw[0];
    *elapsed_ns = t1 - t0;
    return 0;
}

}  // extern "C"
