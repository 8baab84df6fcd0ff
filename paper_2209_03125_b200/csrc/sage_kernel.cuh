// sage_kernel.cuh -- the SCS-2 checksum kernel for sm_100a (product).
//
// One launch = one attestation (SAGE section 5.2.2).  Every logical
// thread of a full-occupancy grid (2048 per SM: 2 CTAs x 1024 threads at 32
// registers, or -- the c2a kernel -- 1 CTA x 1024 threads x 2 lane states at 64 allocated
// registers; the B200 analogue of P:612-613) seeds its state from the nonce, runs R rounds of
// SCS-2 entirely in registers, and the folded states are
// reduced warp (shuffle) -> block (shared memory) -> grid (one 64-bit atomic
// per CTA).
//
// Region placement:
//   SMEM   : the region is copied once per CTA into shared memory with a 1-D
//            TMA bulk copy (cp.async.bulk + mbarrier complete_tx); each round's
//            pick is one LDS.
//   HYBRID : (ADDR 8) the first region_bytes of the region are staged as for
//            SMEM, the rest is read in place; each pick loads from whichever
//            holds it.
//   GLOBAL : each round's pick is one read-only LDG (32/128/256-bit for
//            P = 1/4/8) straight from L2/HBM; the data pointer of the pick is
//            the load address itself.
//
// Integer-pipe mapping (B300_MICROARCH: IMAD on the FMA pipe, LOP3/SHF/IADD3
// on the ALU pipe, 2 cycles per warp instruction each): R7's a*MUL + t is one
// IMAD (FMA pipe) and t = a + rotl(t, S) one LEA.HI-class op (ALU pipe),
// the interleaved shift-and-add pattern of P:651.
//
// This header holds only the product's lowering choices (sage_api.cu picks
// the instantiations).  The measurement knobs of round 1 (timing-adversary
// injections, instruction-mix probes, alternative lowerings, traces) live in
// the bench harness, bench/sage_lab.cuh.
#pragma once
#include <stdint.h>

namespace sage {

constexpr int kAccum = 16;                                   // K
constexpr uint64_t kXsMult = 0x2545F4914F6CDD1DULL;          // xorshift64* multiplier
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;           // SplitMix64 increment

// R7 constant tables (Q6): rotations are compile-time immediates
// (one LEA.HI each); the multipliers reach the kernel through KernelArgs::mul
// (constant bank), see there.
__host__ __device__ constexpr uint32_t mul_of(int j) {
    constexpr uint32_t e[kAccum] = {5, 11, 3, 17, 9, 23, 7, 13, 29, 2, 19, 6, 15, 27, 4, 21};
    return (1u << e[j]) + 1u;
}
__host__ __device__ constexpr uint32_t rot_of(int j) {
    constexpr uint32_t s[kAccum] = {7, 13, 19, 3, 25, 9, 17, 5, 11, 29, 2, 23, 14, 6, 27, 18};
    return s[j];
}

__device__ __forceinline__ uint32_t rotl(uint32_t v, uint32_t s) { return __funnelshift_l(v, v, s); }

__device__ __forceinline__ uint64_t xorshift(uint64_t x) {
    x ^= x >> 12;
    x ^= x << 25;
    x ^= x >> 27;
    return x;
}

__device__ __forceinline__ uint64_t splitmix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// ---- bounds-checked build (test-only: bench/libsage_checked.so, -DSAGE_BOUNDS_CHECK) ----
// Every shared-memory and global address the kernel reads is checked against the
// staged bytes / the region, and a violation traps (the launch fails with an
// error instead of reading out of bounds).  The product build compiles these to
// nothing (tests/test_sass_evidence.py: no trap instruction in libsage.so).
#ifdef SAGE_BOUNDS_CHECK
#define SAGE_CHECK(cond)          \
    do {                          \
        if (!(cond)) __trap();    \
    } while (0)
#else
#define SAGE_CHECK(cond) \
    do {                 \
    } while (0)
#endif

__device__ __forceinline__ uint32_t dynamic_smem_bytes() {
    uint32_t r;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
    return r;
}

// ---- PTX helpers: mbarrier + 1-D TMA bulk copy + read-only loads ------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    while (!done) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    }
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int P> struct Pick { uint32_t w[P]; };

// Read-only global load of one P-word chunk (ld.global.nc: L1-allocating; small,
// L1-resident regions are 6.8x faster than with L1 bypassed).
template <int P>
__device__ __forceinline__ Pick<P> load_global(const uint32_t* p) {
    Pick<P> d;
    uint32_t* w = d.w;
    if constexpr (P == 1) {
        asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(w[0]) : "l"(p));
    } else if constexpr (P == 4) {
        asm volatile("ld.global.nc.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
                     : "l"(p));
    } else {
        asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                     : "l"(p));
    }
    return d;
}

template <int P>
__device__ __forceinline__ Pick<P> load_shared(const uint32_t* s) {
    Pick<P> d;
    if constexpr (P == 1) {
        d.w[0] = *s;
    } else {
#pragma unroll
        for (int h = 0; h < P / 4; ++h) {
            uint4 v = reinterpret_cast<const uint4*>(s)[h];
            d.w[4 * h + 0] = v.x; d.w[4 * h + 1] = v.y; d.w[4 * h + 2] = v.z; d.w[4 * h + 3] = v.w;
        }
    }
    return d;
}

template <int P>
__device__ __forceinline__ Pick<P> load_shared_addr(uint32_t addr) {
    Pick<P> d;
    if constexpr (P == 1) {
        asm volatile("ld.shared.b32 %0, [%1];" : "=r"(d.w[0]) : "r"(addr));
    } else {
#pragma unroll
        for (int h = 0; h < P / 4; ++h)
            asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];"
                         : "=r"(d.w[4 * h]), "=r"(d.w[4 * h + 1]), "=r"(d.w[4 * h + 2]), "=r"(d.w[4 * h + 3])
                         : "r"(addr + 16 * h));
    }
    return d;
}

struct KernelArgs {
    const uint32_t* region;   // device VA of region word 0 (= SCS-2 base)
    uint64_t nonce;
    uint32_t nc_mask;         // Nc - 1
    uint32_t rounds;          // R
    uint32_t region_bytes;    // bytes staged in shared memory (SMEM / HYBRID placement)
    uint64_t* raw;            // [checksum, max cycles, ~min start ns, max end ns]
    uint64_t* per_warp;       // optional, n/32 partial sums
    // R7 multipliers MUL[j] = 2^L[j] + 1, passed through the constant bank so
    // ptxas emits one IMAD R, R, c[..], R per step instead of strength-reducing
    // a*(2^L+1)+t into a*2^L + (a+t) (two FMA-pipe ops).
    uint32_t mul[kAccum];
    uint32_t four_p;          // 4*P as a runtime value (forces IMAD for the chunk offset)
    uint32_t zero;            // 0; operand of the register reservation's result-neutral fold (PAD)
    uint32_t one;             // 1; multiplier that keeps an add on the FMA pipe (ADDR 2/4/8)
    uint32_t* counts;         // COUNT variant only: per-chunk read counters (inclusion experiment)
};

// The region staged in shared memory (SMEM placement): namespace-scope so the
// round can address it with a constant base (LDS [v + const]).
extern __shared__ __align__(128) uint32_t smem_words[];

// SCS-2 R6 / R9 odd multipliers: round index, high DP word, exchanged value.
constexpr uint32_t kKR = 0x9E3779B1u, kKH = 0x85EBCA77u, kKX = 0xC2B2AE3Du;

// One SCS-2 round (R1-R9) for this thread.
//   P        words per pick (1, 4, 8)
//   SMEM     region (or, ADDR 8, its staged prefix) in shared memory, else read from global
//   STRADDLE the region's chunk addresses may differ in their high 32 bits
//            (else hi32(dp) == hi32(base) for every chunk, host-checked)
//   XS       16: y = x * M64 as one wide multiply and two chained IMADs; 0: as ptxas lowers it
//   ADDR     pick addressing of non-straddling SMEM regions:
//            0 generic, 1 chunk offset as IMAD, 2 offsets and the R6 add as IMADs,
//            4 the warp-uniform R6 bracket folded into the chunk-offset IMAD,
//            8 SAGE_HYBRID (staged prefix in shared memory, the rest from global)
//   COUNT    also count reads per chunk into args.counts (the memory-region
//            inclusion experiment); not in the timed path
template <int P, bool SMEM, bool STRADDLE, int XS, int ADDR, bool COUNT>
__device__ __forceinline__ void scs_round(uint32_t (&a)[kAccum], uint32_t& xlo, uint32_t& xhi, uint32_t r,
                                           uint64_t base, uint32_t nc_mask, uint32_t src_lane,
                                           const KernelArgs& args) {
    static_assert(XS == 0 || XS == 16, "product xorshift lowerings");
    static_assert(ADDR == 0 || ADDR == 1 || ADDR == 2 || ADDR == 4 || ADDR == 8, "product pick addressings");
    // R1
    xlo = xlo ^ __funnelshift_r(xlo, xhi, 12);              // x ^= x >> 12
    xhi = xhi ^ (xhi >> 12);
    xhi = xhi ^ __funnelshift_l(xlo, xhi, 25);              // x ^= x << 25
    xlo = xlo ^ (xlo << 25);
    xlo = xlo ^ __funnelshift_r(xlo, xhi, 27);              // x ^= x >> 27
    xhi = xhi ^ (xhi >> 27);
    uint64_t y;
    if constexpr (XS & 16) {
        // y = x * M64 (mod 2^64) as one wide multiply and two chained multiply-adds
        // (3 FMA-pipe ops; ptxas' own lowering uses 4 to shorten the latency)
        uint32_t ylo, yhi;
        asm("{\n\t.reg .u64 w;\n\t"
            "mul.wide.u32 w, %2, %4;\n\t"
            "mov.b64 {%0, %1}, w;\n\t"
            "mad.lo.u32 %1, %2, %5, %1;\n\t"
            "mad.lo.u32 %1, %3, %4, %1;\n\t}"
            : "=&r"(ylo), "=&r"(yhi)
            : "r"(xlo), "r"(xhi), "n"(static_cast<uint32_t>(kXsMult)), "n"(static_cast<uint32_t>(kXsMult >> 32)));
        y = (static_cast<uint64_t>(yhi) << 32) | ylo;
    } else {
        y = ((static_cast<uint64_t>(xhi) << 32) | xlo) * kXsMult;
    }
    // R2, R3
    const uint32_t C = a[kAccum - 1];
    const uint32_t i = (static_cast<uint32_t>(y >> 32) ^ C) & nc_mask;
    if constexpr (COUNT) atomicAdd(&args.counts[i], 1u);
    // bounds-checked build: the region is (nc_mask + 1) chunks of 4P bytes at base;
    // shared memory holds its first args.region_bytes bytes
    const uint64_t region_end = base + (static_cast<uint64_t>(nc_mask) + 1u) * (4u * P);
    (void)region_end;
    // R4, R5, R6 (first part)
    Pick<P> d;
    uint32_t t;
    if constexpr (SMEM && !STRADDLE && ADDR == 4) {
        // as ADDR == 2, with the whole warp-uniform bracket folded into the chunk-offset IMAD
        const uint32_t addr = i * args.four_p + smem_u32(smem_words);
        const uint32_t ur = r * kKR + static_cast<uint32_t>(base) + static_cast<uint32_t>(base >> 32) * kKH;
        SAGE_CHECK(addr - smem_u32(smem_words) + 4u * P <= args.region_bytes);
        d = load_shared_addr<P>(addr);
        t = static_cast<uint32_t>(y) * args.one + (i * args.four_p + ur);
    } else if constexpr (SMEM && !STRADDLE && ADDR == 8) {
        // hybrid placement: chunks below region_bytes are staged in shared memory, the
        // rest is read from global (L1/L2); each lane issues a predicated LDS or LDG for
        // its own pick.  Shared address and 64-bit global address as IMAD / IMAD.WIDE
        // (FMA pipe), the R6 bracket folded as in ADDR == 4.
        const uint32_t saddr = i * args.four_p + smem_u32(smem_words);
        const uint64_t gaddr = static_cast<uint64_t>(i) * args.four_p + base;
        const uint32_t staged_chunks = args.region_bytes / args.four_p;   // loop-invariant
        const uint32_t ur = r * kKR + static_cast<uint32_t>(base) + static_cast<uint32_t>(base >> 32) * kKH;
        SAGE_CHECK(i < staged_chunks ? saddr - smem_u32(smem_words) + 4u * P <= args.region_bytes
                                     : gaddr >= base + args.region_bytes && gaddr + 4u * P <= region_end);
        if constexpr (P == 1) {
            asm volatile("{\n\t.reg .pred p;\n\t"
                         "setp.lt.u32 p, %1, %2;\n\t"
                         "@p ld.shared.b32 %0, [%3];\n\t"
                         "@!p ld.global.nc.b32 %0, [%4];\n\t}"
                         : "=r"(d.w[0]) : "r"(i), "r"(staged_chunks), "r"(saddr), "l"(gaddr));
        } else if constexpr (P == 4) {
            asm volatile("{\n\t.reg .pred p;\n\t"
                         "setp.lt.u32 p, %4, %5;\n\t"
                         "@p ld.shared.v4.b32 {%0,%1,%2,%3}, [%6];\n\t"
                         "@!p ld.global.nc.v4.b32 {%0,%1,%2,%3}, [%7];\n\t}"
                         : "=r"(d.w[0]), "=r"(d.w[1]), "=r"(d.w[2]), "=r"(d.w[3])
                         : "r"(i), "r"(staged_chunks), "r"(saddr), "l"(gaddr));
        } else {
            static_assert(P == 8, "one, four or eight words per pick");
            asm volatile("{\n\t.reg .pred p;\n\t"
                         "setp.lt.u32 p, %8, %9;\n\t"
                         "@p ld.shared.v4.b32 {%0,%1,%2,%3}, [%10];\n\t"
                         "@p ld.shared.v4.b32 {%4,%5,%6,%7}, [%10+16];\n\t"
                         "@!p ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%11];\n\t}"
                         : "=r"(d.w[0]), "=r"(d.w[1]), "=r"(d.w[2]), "=r"(d.w[3]),
                           "=r"(d.w[4]), "=r"(d.w[5]), "=r"(d.w[6]), "=r"(d.w[7])
                         : "r"(i), "r"(staged_chunks), "r"(saddr), "l"(gaddr));
        }
        t = static_cast<uint32_t>(y) * args.one + (i * args.four_p + ur);
    } else if constexpr (SMEM && !STRADDLE && ADDR == 2) {
        // both chunk offsets and the R6 add as IMADs (FMA pipe), sparing the ALU pipe
        const uint32_t addr = i * args.four_p + smem_u32(smem_words);
        const uint32_t lo_dp = i * args.four_p + static_cast<uint32_t>(base);
        SAGE_CHECK(addr - smem_u32(smem_words) + 4u * P <= args.region_bytes);
        d = load_shared_addr<P>(addr);
        t = static_cast<uint32_t>(y) * args.one + lo_dp + (r * kKR + static_cast<uint32_t>(base >> 32) * kKH);
    } else if constexpr (SMEM && !STRADDLE && ADDR == 1) {
        // shared-window address of the chunk on the FMA pipe; lo32(dp) = addr + (lo32(base) - smem)
        const uint32_t addr = i * args.four_p + smem_u32(smem_words);
        SAGE_CHECK(addr - smem_u32(smem_words) + 4u * P <= args.region_bytes);
        d = load_shared_addr<P>(addr);
        const uint32_t base_minus_smem = static_cast<uint32_t>(base) - smem_u32(smem_words);   // loop-invariant
        // lo32(y) + r*KR + lo32(dp) + hi32(dp)*KH with lo32(dp) = addr + base_minus_smem; the bracket is
        // warp-uniform (uniform datapath)
        t = static_cast<uint32_t>(y) + (r * kKR + base_minus_smem + static_cast<uint32_t>(base >> 32) * kKH) + addr;
    } else if constexpr (SMEM && !STRADDLE) {
        const uint32_t v = i * (4u * P);                         // byte offset of the chunk
        SAGE_CHECK(v + 4u * P <= args.region_bytes);
        d = load_shared<P>(smem_words + static_cast<size_t>(i) * P);
        t = static_cast<uint32_t>(y) + (r * kKR + static_cast<uint32_t>(base) + static_cast<uint32_t>(base >> 32) * kKH) + v;
    } else {
        const uint64_t dp = base + static_cast<uint64_t>(i) * (4u * P);   // R5 (= the global load address)
        SAGE_CHECK(SMEM ? (static_cast<uint64_t>(i) + 1u) * (4u * P) <= args.region_bytes
                        : dp >= base && dp + 4u * P <= region_end);
        if constexpr (SMEM) d = load_shared<P>(smem_words + static_cast<size_t>(i) * P);
        else d = load_global<P>(reinterpret_cast<const uint32_t*>(dp));
        t = static_cast<uint32_t>(y) + r * kKR + static_cast<uint32_t>(dp) + static_cast<uint32_t>(dp >> 32) * kKH;
    }
    // R6 (data)
#pragma unroll
    for (int q = 0; q < P; ++q) t = rotl(t, 5) + d.w[q];
    // R7
#pragma unroll
    for (int j = 0; j < kAccum; ++j) {
        a[j] = a[j] * args.mul[j] + t;
        t = a[j] + rotl(t, rot_of(j));
    }
    // R8
    t = t + (t >> (C & 31u));
    // R9 (SCS-2: multiply-add exchange)
    a[kAccum - 1] = a[kAccum - 1] * kKX + __shfl_sync(0xFFFFFFFFu, t, src_lane);
}

// The checksum kernel (one attestation per launch).
//   UNROLL   rounds per trip of the round loop (remainder rounds run one by one)
//   ILP      logical SCS-2 warps per hardware warp: 1 = one lane state per
//            thread, 2 CTAs x 1024 threads per SM at 32 registers; 2 = two
//            independent lane states per thread (interleaved by ptxas), one
//            CTA x 1024 threads per SM at 57-64 registers (64 allocated) -- the same register file
//            and logical grid, but all 32 warps of the SM progress together.
//   PAD      registers reserved (kept live across the round loop, unused) so that
//            an ILP > 1 kernel allocates the whole register file
// UNROLL and PAD do not change the arithmetic; they steer ptxas' schedule
// (schedule search).
template <int P, bool SMEM, bool STRADDLE, int XS, int UNROLL, int ADDR, bool COUNT = false, int ILP = 1, int PAD = 0>
__global__ void __launch_bounds__(1024, ILP == 1 ? 2 : 1) sage_checksum_kernel(const KernelArgs args) {
    static_assert(ILP == 1 || ILP == 2, "one or two lane states per thread");
    __shared__ uint64_t red[32];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint64_t t_start_ns;
    __shared__ long long c_start;

    // a13: CTA start time (kept in shared memory, not in registers)
    if (threadIdx.x == 0) {
        t_start_ns = globaltimer();
        c_start = clock64();
    }

    // a2: stage the region (or its prefix, HYBRID) into shared memory.
    if constexpr (SMEM) {
        const uint32_t bytes = args.region_bytes;
        SAGE_CHECK(bytes <= dynamic_smem_bytes() &&
                   bytes <= (static_cast<uint64_t>(args.nc_mask) + 1u) * (4u * P) && bytes % (4u * P) == 0);
        if ((bytes & 15u) == 0) {
            if (threadIdx.x == 0) mbar_init(&bar, 1);
            __syncthreads();
            if (threadIdx.x == 0) {
                mbar_expect_tx(&bar, bytes);
                constexpr uint32_t kChunk = 32768;
                for (uint32_t off = 0; off < bytes; off += kChunk) {
                    const uint32_t n = (bytes - off < kChunk) ? (bytes - off) : kChunk;
                    bulk_g2s(reinterpret_cast<char*>(smem_words) + off, reinterpret_cast<const char*>(args.region) + off,
                             n, &bar);
                }
            }
            mbar_wait(&bar, 0);
        } else {  // 4- or 8-byte regions: below the bulk-copy granule
            for (uint32_t k = threadIdx.x; k < bytes / 4; k += blockDim.x) smem_words[k] = args.region[k];
            __syncthreads();
        }
    }

    // a1: I1-I3.  Hardware warp hw computes the ILP logical SCS-2 warps
    // hw*ILP .. hw*ILP+ILP-1 (lane l of each); logical thread g = 32*warp + l.
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t src_lane = (lane + 1u) & 31u;
    const uint32_t warp = threadIdx.x >> 5;
    const uint64_t hw_warp = static_cast<uint64_t>(blockIdx.x) * (blockDim.x >> 5) + warp;
    uint32_t a[ILP][kAccum];
    uint32_t xlo[ILP], xhi[ILP];
#pragma unroll
    for (int s = 0; s < ILP; ++s) {
        const uint64_t g = (hw_warp * ILP + s) * 32u + lane;
        uint64_t x = splitmix(args.nonce + (g + 1) * kGamma);
        if (x == 0) x = kGamma;
#pragma unroll
        for (int j = 0; j < kAccum; ++j) {
            x = xorshift(x);
            a[s][j] = static_cast<uint32_t>((x * kXsMult) >> 32);
        }
        xlo[s] = static_cast<uint32_t>(x);
        xhi[s] = static_cast<uint32_t>(x >> 32);
    }

    // PAD: register reservation -- PAD per-lane values from %clock (not recomputable)
    // before the round loop and consumed after it, so they stay in registers for
    // the whole attestation and the CTA's register allocation grows by PAD
    uint32_t pad[PAD > 0 ? PAD : 1];
    if constexpr (PAD > 0) {
#pragma unroll
        for (int k = 0; k < PAD; ++k)          // per-lane values, so they occupy vector registers
            asm volatile("{\n\t.reg .b32 c;\n\tmov.u32 c, %%clock;\n\tmov.u32 %0, %%laneid;\n\t"
                         "add.u32 %0, %0, c;\n\t}" : "=r"(pad[k]));
    }

    const uint64_t base = reinterpret_cast<uint64_t>(args.region);
    const uint32_t nc_mask = args.nc_mask;
    const uint32_t rounds = args.rounds;

    // a10: round loop, UNROLL rounds (of every lane state) per trip + remainder
    uint32_t r = 0;
    const uint32_t main_end = rounds - rounds % UNROLL;
    for (; r < main_end; r += UNROLL) {
#pragma unroll
        for (int uu = 0; uu < UNROLL * ILP; ++uu) {
            const int u = uu / ILP;                     // round-major: (u, s)
            const int s = uu % ILP;
            scs_round<P, SMEM, STRADDLE, XS, ADDR, COUNT>(a[s], xlo[s], xhi[s], r + u, base, nc_mask, src_lane, args);
        }
    }
    for (; r < rounds; ++r) {
#pragma unroll
        for (int s = 0; s < ILP; ++s)
            scs_round<P, SMEM, STRADDLE, XS, ADDR, COUNT>(a[s], xlo[s], xhi[s], r, base, nc_mask, src_lane, args);
    }

    if constexpr (PAD > 0) {
#pragma unroll
        for (int k = 0; k < PAD; ++k)          // xlo ^= pad & 0 (args.zero): result-neutral
            asm volatile("{\n\t.reg .b32 q;\n\tand.b32 q, %1, %2;\n\txor.b32 %0, %0, q;\n\t}"
                         : "+r"(xlo[0]) : "r"(pad[k]), "r"(args.zero));
    }

    // a11: F1-F2, a12: warp -> block -> grid
    uint64_t fw = 0;
#pragma unroll
    for (int s = 0; s < ILP; ++s) {
        uint32_t e = 0, o = 0;
#pragma unroll
        for (int j = 0; j < kAccum; j += 2) { e ^= a[s][j]; o ^= a[s][j + 1]; }
        uint64_t f = ((static_cast<uint64_t>(o) << 32) | e) ^ ((static_cast<uint64_t>(xhi[s]) << 32) | xlo[s]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) f += __shfl_down_sync(0xFFFFFFFFu, f, off);
        if (lane == 0 && args.per_warp) args.per_warp[hw_warp * ILP + s] = f;
        fw += f;
    }
    if (lane == 0) red[warp] = fw;
    __syncthreads();
    if (warp == 0) {
        const uint32_t nw = blockDim.x >> 5;
        uint64_t s = (lane < nw) ? red[lane] : 0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xFFFFFFFFu, s, off);
        if (lane == 0) {
            // a13: timing
            const long long c_end = clock64();
            const uint64_t t_end_ns = globaltimer();
            atomicAdd(reinterpret_cast<unsigned long long*>(&args.raw[0]), static_cast<unsigned long long>(s));
            atomicMax(reinterpret_cast<unsigned long long*>(&args.raw[1]),
                      static_cast<unsigned long long>(c_end - c_start));
            atomicMax(reinterpret_cast<unsigned long long*>(&args.raw[2]),
                      static_cast<unsigned long long>(~t_start_ns));
            atomicMax(reinterpret_cast<unsigned long long*>(&args.raw[3]),
                      static_cast<unsigned long long>(t_end_ns));
        }
    }
}

// Host-side helper: fill the constant-bank tables of KernelArgs.
inline void fill_tables(KernelArgs& args, uint32_t P) {
    args.four_p = 4u * P;
    args.zero = 0;
    args.one = 1;
    for (int j = 0; j < kAccum; ++j) args.mul[j] = mul_of(j);
}

}  // namespace sage
