// microbench.cu -- L0 probes for the integer-pipe roofline.
//
// Each probe runs at full occupancy (2 CTAs x 1024 threads per SM, <= 32 regs)
// a loop of independent dependency chains of one SASS op class, and reports
// warp-instructions issued per SM per cycle (clock64 around the loop, max over
// CTAs) -- i.e. the measured issue rate of that op class on sm_100a.  Also a
// random SMEM gather and a dependent random HBM gather at full occupancy.
// Output: one JSON line per probe.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e = (x);                                                   \
        if (e != cudaSuccess) {                                                \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));            \
            exit(1);                                                           \
        }                                                                      \
    } while (0)

struct Args {
    uint32_t iters;
    uint32_t c0, c1, c2, c3;   // runtime constants (defeat strength reduction)
    unsigned long long* cycles;
    uint32_t* sink;
};

constexpr int CH = 8;   // independent chains per thread

#define PROBE(NAME, BODY)                                                          \
    __global__ void __launch_bounds__(1024, 2) NAME(Args a) {                      \
        uint32_t v[CH];                                                            \
        _Pragma("unroll") for (int k = 0; k < CH; ++k) v[k] = threadIdx.x * (k + 3) + a.c3; \
        __syncthreads();                                                           \
        long long t0 = clock64();                                                  \
        _Pragma("unroll 1") for (uint32_t it = 0; it < a.iters; ++it) {             \
            _Pragma("unroll") for (int u = 0; u < 4; ++u) {                        \
                _Pragma("unroll") for (int k = 0; k < CH; ++k) { BODY; }           \
            }                                                                      \
        }                                                                          \
        __syncthreads();                                                           \
        long long t1 = clock64();                                                  \
        uint32_t s = 0;                                                            \
        _Pragma("unroll") for (int k = 0; k < CH; ++k) s ^= v[k];                  \
        if (s == 0x12345679u) a.sink[0] = s;                                       \
        if (threadIdx.x == 0) atomicMax(a.cycles, (unsigned long long)(t1 - t0));  \
    }

// IMAD with a constant-bank multiplier: v = v * c0 + c1      (FMA pipe)
PROBE(p_imad, v[k] = v[k] * v[(k + 1) & (CH - 1)] + a.c1)
// LOP3: v = v ^ (v >> 0)... use a 3-input logic op on registers (ALU pipe)
PROBE(p_lop3, asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(v[k]) : "r"(a.c0), "r"(a.c1)))
// IADD3
PROBE(p_iadd3, v[k] = v[k] + v[(k + 1) & (CH - 1)] + a.c1)
// SHF (funnel shift by immediate)
PROBE(p_shf, v[k] = __funnelshift_l(v[k], v[k], 7))
// LEA.HI-form: v = c + rotl(v, 7)
PROBE(p_leahi, v[k] = a.c0 + __funnelshift_l(v[k], v[k], 7))
// IMAD.WIDE.U32: 64-bit product, keep both halves
// multiply-with-carry on a 64-bit chain pair: one IMAD.WIDE.U32 lo, c, {hi} per body
PROBE(p_imadwide, { if (k < CH / 2) { unsigned long long w = ((unsigned long long)v[2 * k + 1] << 32) | v[2 * k];
                    w = (unsigned long long)v[2 * k] * a.c0 + (w >> 32); v[2 * k] = (uint32_t)w; v[2 * k + 1] = (uint32_t)(w >> 32); } })
// IMAD.HI.U32
PROBE(p_imadhi, v[k] = __umulhi(v[k], v[(k + 1) & (CH - 1)]) + a.c1)
// 1:1 IMAD + LEA.HI (the R7 pattern)
PROBE(p_mix11, { v[k] = v[k] * a.c0 + a.c1; v[k] = a.c2 + __funnelshift_l(v[k], v[k], 7); })

__global__ void __launch_bounds__(1024, 2) p_smem_gather(Args a) {
    __shared__ uint32_t s[8192];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) s[i] = i * 2654435761u;
    __syncthreads();
    uint32_t x = threadIdx.x * 0x9E3779B9u + a.c3;
    long long t0 = clock64();
    for (uint32_t it = 0; it < a.iters * 4; ++it) {
        x = x * 1664525u + 1013904223u;
        x += s[x >> 19];
    }
    __syncthreads();
    long long t1 = clock64();
    if (x == 0x12345679u) a.sink[0] = x;
    if (threadIdx.x == 0) atomicMax(a.cycles, (unsigned long long)(t1 - t0));
}

__global__ void __launch_bounds__(1024, 2) p_hbm_gather(Args a, const uint32_t* __restrict__ buf, uint32_t mask) {
    uint32_t x = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B9u + a.c3;
    long long t0 = clock64();
    for (uint32_t it = 0; it < a.iters; ++it) {
        x = x * 1664525u + 1013904223u;
        uint32_t w;
        asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(w) : "l"(buf + ((x >> 3) & mask) * 8u));
        x ^= w;
    }
    long long t1 = clock64();
    if (x == 0x12345679u) a.sink[0] = x;
    if (threadIdx.x == 0) atomicMax(a.cycles, (unsigned long long)(t1 - t0));
}

// MLP-k dependent random gathers: k independent chains per thread, one 4-B load
// per 32-B sector, over `mask+1` sectors.  Tells whether random HBM reads are
// latency-bound (rate grows with k) or transaction-bound (flat in k).
// OP: cache operator of the load -- 0 ld.global.nc (L1-allocating read-only),
// 1 ld.global.nc.L1::no_allocate, 2 ld.global.cg (L2 only), 3 ld.global.ca (round 2).
template <int OP>
__device__ __forceinline__ uint32_t gather_load(const uint32_t* p) {
    uint32_t w;
    if constexpr (OP == 0) asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(w) : "l"(p));
    else if constexpr (OP == 1) asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(w) : "l"(p));
    else if constexpr (OP == 2) asm volatile("ld.global.cg.b32 %0, [%1];" : "=r"(w) : "l"(p));
    else asm volatile("ld.global.ca.b32 %0, [%1];" : "=r"(w) : "l"(p));
    return w;
}

template <int K, int OP = 0>
__global__ void __launch_bounds__(1024, 2) p_hbm_gather_mlp(Args a, const uint32_t* __restrict__ buf, uint32_t mask) {
    uint32_t x[K];
#pragma unroll
    for (int k = 0; k < K; ++k) x[k] = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B9u + a.c3 + 77u * k;
    for (uint32_t it = 0; it < a.iters; ++it) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            x[k] = x[k] * 1664525u + 1013904223u;
            const uint32_t w = gather_load<OP>(buf + ((x[k] >> 3) & mask) * 8u);
            x[k] ^= w;
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) s ^= x[k];
    if (s == 0x12345679u) a.sink[0] = s;
}

int gather_only(size_t mb, int op) {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    Args a{};
    a.c3 = 7;
    CK(cudaMalloc(&a.sink, 4));
    size_t bytes = mb << 20;
    uint32_t* buf = nullptr;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMemset(buf, 1, bytes));
    uint32_t mask = uint32_t(bytes / 32 - 1);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    a.iters = 2048;
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        CK(cudaEventRecord(e0));
        void (*fns[])(Args, const uint32_t*, uint32_t) = {p_hbm_gather_mlp<1, 0>, p_hbm_gather_mlp<1, 1>,
                                                          p_hbm_gather_mlp<1, 2>, p_hbm_gather_mlp<1, 3>};
        fns[op & 3]<<<2 * sms, 1024>>>(a, buf, mask);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
    }
    double picks = double(2 * sms) * 1024 * a.iters;
    printf("{\"probe\": \"hbm_gather_mlp\", \"mib\": %zu, \"mlp\": 1, \"op\": %d, \"picks_per_s\": %.4e, \"ms\": %.3f}\n",
           mb, op, picks / (best * 1e-3), best);
    return 0;
}

// Dependent random-sector gather over an L2-resident window (round 2, session 3):
// the MLP-1 chain of p_hbm_gather_mlp, but each pick is one 4-B load from a
// random 32-B sector of [skip, skip + span) inside a buffer of `total` bytes
// (non-power-of-two spans by a multiply-high range reduction).  With
// total = 524,288 and skip = 192 KiB this is the in-place part of the paper's
// buffer under SAGE_HYBRID -- every pick an L1 miss to an L2 hit, no checksum
// arithmetic: the measured ceiling of the L1->L2 request path for that pattern
// (bench.py's c2c / c2cp4 / c2cp8 roofline records).  Geometry as the hybrid
// kernel: one CTA x 1024 threads x 2 chains per SM, 192 KiB shared memory reserved.
template <int OP>
__global__ void __launch_bounds__(1024, 1) p_l2_gather(Args a, const uint32_t* __restrict__ buf, uint32_t nsect) {
    // two independent chains per thread, one CTA of 1024 threads per SM: the
    // SAGE_HYBRID kernel's geometry (two lane states per thread)
    uint32_t x0 = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B9u + a.c3, x1 = x0 ^ 0x85EBCA77u;
    for (uint32_t it = 0; it < a.iters; ++it) {
        x0 = x0 * 1664525u + 1013904223u;
        x1 = x1 * 1664525u + 1013904223u;
        const uint32_t w0 = gather_load<OP>(buf + __umulhi(x0, nsect) * 8u);
        const uint32_t w1 = gather_load<OP>(buf + __umulhi(x1, nsect) * 8u);
        x0 ^= w0;
        x1 ^= w1;
    }
    if ((x0 ^ x1) == 0x12345679u) a.sink[0] = x0;
}

int l2_gather(size_t total, size_t skip, int op) {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    if (skip >= total || total % 32 || skip % 32) { fprintf(stderr, "need 0 <= skip < total, multiples of 32\n"); return 1; }
    Args a{};
    a.c3 = 7;
    CK(cudaMalloc(&a.sink, 4));
    uint32_t* buf = nullptr;
    CK(cudaMalloc(&buf, total));
    CK(cudaMemset(buf, 1, total));
    const uint32_t nsect = uint32_t((total - skip) / 32);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    a.iters = 16384;   // ~20 ms per launch: long enough for the clocks to settle
    void (*fns[])(Args, const uint32_t*, uint32_t) = {p_l2_gather<0>, p_l2_gather<1>, p_l2_gather<2>, p_l2_gather<3>};
    // the same shared-memory carve-out as the hybrid kernel: 192 KiB of dynamic shared
    // memory per CTA (unused), which leaves L1 the rest of the SM's 256 KB
    const int dyn = 192 * 1024;
    CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(fns[op & 3]), cudaFuncAttributeMaxDynamicSharedMemorySize, dyn));
    float best = 1e30f;
    for (int rep = 0; rep < 12; ++rep) {   // the first launches ramp an idle GPU's clocks
        CK(cudaEventRecord(e0));
        fns[op & 3]<<<sms, 1024, dyn>>>(a, buf + skip / 4, nsect);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (rep >= 4 && ms < best) best = ms;
    }
    const double picks = double(sms) * 1024 * 2 * a.iters;
    int clk_khz = 0;
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
    printf("{\"probe\": \"l2_gather\", \"total_bytes\": %zu, \"skip_bytes\": %zu, \"op\": %d, "
           "\"picks_per_s\": %.4e, \"picks_per_sm_clk_at_max\": %.4f, \"ms\": %.3f}\n",
           total, skip, op, picks / (best * 1e-3), picks / (best * 1e-3) / sms / (clk_khz * 1e3), best);
    return 0;
}

// Concurrency sweep of the dependent random-sector gather (round 2, session 2):
// the same MLP-1 probe over a power-of-two buffer with 1 .. 2048 chains per SM
// (blocks = SMs or 2 x SMs, 32 .. 1024 threads).  Little's law gives the mean
// latency per pick, concurrency / rate: a rate that stops growing while the
// latency grows with the concurrency is a throughput limit in the memory system
// (queueing), not a latency limit.
int gather_concurrency(size_t mb) {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    Args a{};
    a.c3 = 7;
    CK(cudaMalloc(&a.sink, 4));
    size_t bytes = mb << 20;
    if (bytes & (bytes - 1)) { fprintf(stderr, "power-of-two MiB only\n"); return 1; }
    uint32_t* buf = nullptr;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMemset(buf, 1, bytes));
    const uint32_t mask = uint32_t(bytes / 32 - 1);
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const int shapes[][2] = {{1, 32}, {1, 64}, {1, 128}, {1, 256}, {1, 512}, {1, 1024}, {2, 1024}};
    for (auto& sh : shapes) {
        const int blocks = sh[0] * sms, threads = sh[1];
        a.iters = threads >= 512 ? 2048 : 4096;
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaEventRecord(e0));
            p_hbm_gather_mlp<1, 0><<<blocks, threads>>>(a, buf, mask);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < best) best = ms;
        }
        const double conc = double(blocks) * threads, picks = conc * a.iters, rate = picks / (best * 1e-3);
        printf("{\"probe\": \"hbm_gather_concurrency\", \"mib\": %zu, \"chains_per_sm\": %d, \"concurrency\": %.0f, "
               "\"picks_per_s\": %.4e, \"little_latency_ns\": %.1f, \"ms\": %.3f}\n",
               mb, blocks / sms * threads, conc, rate, 1e9 * conc / rate, best);
        fflush(stdout);
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 2 && strcmp(argv[1], "gather") == 0)
        return gather_only(strtoull(argv[2], nullptr, 10), argc > 3 ? atoi(argv[3]) : 0);
    if (argc > 3 && strcmp(argv[1], "l2gather") == 0)
        return l2_gather(strtoull(argv[2], nullptr, 10), strtoull(argv[3], nullptr, 10), argc > 4 ? atoi(argv[4]) : 0);
    if (argc > 2 && strcmp(argv[1], "conc") == 0)
        return gather_concurrency(strtoull(argv[2], nullptr, 10));
    int dev = 0, sms = 0, clk = 0;
    CK(cudaSetDevice(dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
    Args a{};
    a.c0 = 33; a.c1 = 0x9E3779B9u; a.c2 = 12345; a.c3 = 7;
    CK(cudaMalloc(&a.cycles, 8));
    CK(cudaMalloc(&a.sink, 4));
    const int blocks = 2 * sms, threads = 1024, warps_per_sm = 64;
    struct P { const char* name; void (*fn)(Args); int ops_per_body; };
    P probes[] = {{"imad_const", p_imad, 1}, {"lop3", p_lop3, 1}, {"iadd", p_iadd3, 1}, {"shf_funnel", p_shf, 1},
                  {"lea_hi_form", p_leahi, 1}, {"imad_wide_u32+iadd3", p_imadwide, -16}, {"imad_hi_u32", p_imadhi, 1},
                  {"imad+lea_hi", p_mix11, 2}};
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (auto& p : probes) {
        a.iters = 4096;
        for (int rep = 0; rep < 2; ++rep) {
            CK(cudaMemset(a.cycles, 0, 8));
            CK(cudaEventRecord(e0));
            p.fn<<<blocks, threads>>>(a);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
        }
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        unsigned long long cyc = 0;
        CK(cudaMemcpy(&cyc, a.cycles, 8, cudaMemcpyDeviceToHost));
        // per thread; a negative ops_per_body means that many bodies per iteration
        double bodies = double(a.iters) * (p.ops_per_body < 0 ? -p.ops_per_body : 4 * CH);
        double warp_bodies_per_sm_cycle = bodies * warps_per_sm / double(cyc);
        double eff_mhz = double(cyc) / (ms * 1e3);
        printf("{\"probe\": \"%s\", \"warp_bodies_per_sm_clk\": %.4f, \"src_ops_per_body\": %d, \"cycles\": %llu, "
               "\"ms\": %.4f, \"eff_mhz\": %.1f}\n",
               p.name, warp_bodies_per_sm_cycle, p.ops_per_body, cyc, ms, eff_mhz);
    }
    {   // random SMEM gather, 32 KiB table: LCG (IMAD) + shift + LDS + add per body
        a.iters = 4096;
        for (int rep = 0; rep < 2; ++rep) {
            CK(cudaMemset(a.cycles, 0, 8));
            CK(cudaEventRecord(e0));
            p_smem_gather<<<blocks, threads>>>(a);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
        }
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        unsigned long long cyc = 0;
        CK(cudaMemcpy(&cyc, a.cycles, 8, cudaMemcpyDeviceToHost));
        double bodies = double(a.iters) * 4;
        printf("{\"probe\": \"smem_random_gather\", \"warp_bodies_per_sm_clk\": %.4f, \"cycles\": %llu, \"ms\": %.4f}\n",
               bodies * warps_per_sm / double(cyc), cyc, ms);
    }
    for (size_t gib : {1, 4}) {   // dependent random 4-B loads, one per 32-B sector, over gib GiB
        size_t bytes = gib << 30;
        uint32_t* buf = nullptr;
        CK(cudaMalloc(&buf, bytes));
        CK(cudaMemset(buf, 1, bytes));
        uint32_t mask = uint32_t(bytes / 32 - 1);
        a.iters = 2048;
        for (int rep = 0; rep < 2; ++rep) {
            CK(cudaMemset(a.cycles, 0, 8));
            CK(cudaEventRecord(e0));
            p_hbm_gather<<<blocks, threads>>>(a, buf, mask);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
        }
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        double picks = double(blocks) * threads * a.iters;
        printf("{\"probe\": \"hbm_dependent_sector_gather\", \"gib\": %zu, \"picks_per_s\": %.4e, "
               "\"sector_gbps\": %.1f, \"ms\": %.3f}\n", gib, picks / (ms * 1e-3), picks * 32 / (ms * 1e-3) / 1e9, ms);
        CK(cudaFree(buf));
    }
    for (size_t mb : {256, 2048}) {
        size_t bytes = mb << 20;
        uint32_t* buf = nullptr;
        CK(cudaMalloc(&buf, bytes));
        CK(cudaMemset(buf, 1, bytes));
        uint32_t mask = uint32_t(bytes / 32 - 1);
        void (*fns[])(Args, const uint32_t*, uint32_t) = {p_hbm_gather_mlp<1>, p_hbm_gather_mlp<2>, p_hbm_gather_mlp<4>};
        int ks[] = {1, 2, 4};
        for (int f = 0; f < 3; ++f) {
            a.iters = 2048 / ks[f];
            float ms = 0;
            for (int rep = 0; rep < 2; ++rep) {
                CK(cudaEventRecord(e0));
                fns[f]<<<blocks, threads>>>(a, buf, mask);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
            }
            CK(cudaEventElapsedTime(&ms, e0, e1));
            double picks = double(blocks) * threads * a.iters * ks[f];
            printf("{\"probe\": \"hbm_gather_mlp\", \"mib\": %zu, \"mlp\": %d, \"picks_per_s\": %.4e, \"ms\": %.3f}\n",
                   mb, ks[f], picks / (ms * 1e-3), ms);
        }
        CK(cudaFree(buf));
    }
    return 0;
}
