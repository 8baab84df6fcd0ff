// sage_lab.cuh -- the experiment ("lab") form of the SCS-2 checksum kernel.
//
// NOT PRODUCT CODE.  This is the round-1 kernel template with every
// measurement knob (EXTRA/EVERY/FEXTRA timing-adversary injections, PROBE
// instruction-mix probes, SYNC barriers, LD cache policies, the ADDR 3/5/6/7
// lowering alternatives, the XS 1/2/4/8 IMAD.WIDE xorshift forms, diagnostic
// traces), kept in the bench harness so the measurements under
// profiles/r01/variants/ and the adversary experiments stay reproducible
// (bench/variants.cu, bench/adversary*.cu, bench/cta_trace.cu,
// bench/stall_trace.cu).  The product kernel is
// paper_2209_03125_b200/csrc/sage_kernel.cuh: the same round with only the
// product's lowering choices.  tests/test_sass_evidence.py checks that this
// template, instantiated with the product's parameters and every knob off,
// compiles to the same instruction sequence as the product kernel, so a lab
// adversary is "the product plus its injection".
//
// Extra lab-only state (LabArgs) follows the product's KernelArgs fields.
//
// (Original header of the round-1 kernel follows.)
//
// sage_kernel.cuh -- the SCS-2 checksum kernel for sm_100a.
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
//   GLOBAL : each round's pick is one read-only LDG (32/128/256-bit for
//            P = 1/4/8) straight from L2/HBM; the data pointer of the pick is
//            the load address itself.
//
// Integer-pipe mapping (B300_MICROARCH: IMAD on the FMA pipe, LOP3/SHF/IADD3
// on the ALU pipe, 2 cycles per warp instruction each): R7's a*MUL + t is one
// IMAD (FMA pipe) and t = a + rotl(t, S) one LEA.HI-class op (ALU pipe),
// the interleaved shift-and-add pattern of P:651.
//
// Template knobs of sage_checksum_kernel.  The product (sage_api.cu) uses
// LD=0, EXTRA=0, COUNT=false (except sage_attest_coverage), ILP=1;
// XS=16 for P=1 SMEM and for every GLOBAL kernel (XS=0 otherwise); and
// ADDR=4 (P=1) / ADDR=2 (P=4) / ADDR=1 (P=8) for non-straddling SMEM regions;
// the other values are lowering alternatives measured by bench/variants.cu and
// bench/adversary.cu and kept so those measurements stay reproducible
// (DESIGN.md section 8).
#pragma once
#include <stdint.h>

namespace sage_lab {

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

// Read-only global loads of one P-word chunk.  LD selects the cache policy:
//   0: ld.global.nc                          (L1-allocating; small, L1-resident regions)
//   1: ld.global.nc.L1::no_allocate          (no L1 allocation)
//   2: ld.global.cg                          (cache at L2 only)
//   3: ld.global.nc.L2::64B                  (64-B L2 fetch hint)
//   4: ld.global.nc.L1::no_allocate.L2::cache_hint with an evict_first policy
//   5: ld.global.nc.L2::cache_hint, policy per pick: evict_last for chunks below
//      args.persist_bytes, evict_first above (round 2: L2 residency for HBM regions)
//   6: as 5 with evict_normal instead of evict_first above persist_bytes
template <int P, int LD>
__device__ __forceinline__ Pick<P> load_global(const uint32_t* p, uint64_t policy) {
    Pick<P> d;
    uint32_t* w = d.w;
    if constexpr (P == 1) {
        if constexpr (LD == 0) asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(w[0]) : "l"(p));
        else if constexpr (LD == 1) asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(w[0]) : "l"(p));
        else if constexpr (LD == 2) asm volatile("ld.global.cg.b32 %0, [%1];" : "=r"(w[0]) : "l"(p));
        else if constexpr (LD == 3) asm volatile("ld.global.nc.L2::64B.b32 %0, [%1];" : "=r"(w[0]) : "l"(p));
        else if constexpr (LD >= 5) asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(w[0]) : "l"(p), "l"(policy));
        else asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(w[0]) : "l"(p), "l"(policy));
    } else if constexpr (P == 4) {
#define O4 "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3])
        if constexpr (LD == 0) asm volatile("ld.global.nc.v4.b32 {%0,%1,%2,%3}, [%4];" : O4 : "l"(p));
        else if constexpr (LD == 1) asm volatile("ld.global.nc.L1::no_allocate.v4.b32 {%0,%1,%2,%3}, [%4];" : O4 : "l"(p));
        else if constexpr (LD == 2) asm volatile("ld.global.cg.v4.b32 {%0,%1,%2,%3}, [%4];" : O4 : "l"(p));
        else if constexpr (LD == 3) asm volatile("ld.global.nc.L2::64B.v4.b32 {%0,%1,%2,%3}, [%4];" : O4 : "l"(p));
        else if constexpr (LD >= 5) asm volatile("ld.global.nc.L2::cache_hint.v4.b32 {%0,%1,%2,%3}, [%4], %5;" : O4 : "l"(p), "l"(policy));
        else asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.b32 {%0,%1,%2,%3}, [%4], %5;" : O4 : "l"(p), "l"(policy));
#undef O4
    } else {
#define O8 "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
        if constexpr (LD == 0) asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : O8 : "l"(p));
        else if constexpr (LD == 1) asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : O8 : "l"(p));
        else if constexpr (LD == 2) asm volatile("ld.global.cg.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : O8 : "l"(p));
        else if constexpr (LD == 3) asm volatile("ld.global.nc.L2::64B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : O8 : "l"(p));
        else if constexpr (LD >= 5) asm volatile("ld.global.nc.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;" : O8 : "l"(p), "l"(policy));
        else asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;" : O8 : "l"(p), "l"(policy));
#undef O8
    }
    return d;
}

__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint64_t evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint64_t evict_normal_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
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
    uint32_t region_bytes;    // SMEM staging size (SMEM placement only)
    uint64_t* raw;            // [checksum, max cycles, ~min start ns, max end ns]
    uint64_t* per_warp;       // optional, n/32 partial sums
    // R7 multipliers MUL[j] = 2^L[j] + 1, passed through the constant bank so
    // ptxas emits one IMAD R, R, c[..], R per step instead of strength-reducing
    // a*(2^L+1)+t into a*2^L + (a+t) (two FMA-pipe ops).
    uint32_t mul[kAccum];
    // 2^20, 2^25, 2^5: xorshift shift multipliers for the IMAD.WIDE lowering
    // (constant bank, so ptxas cannot turn them back into ALU shifts).
    uint32_t p2[3];
    uint32_t four_p;          // 4*P as a runtime value (forces IMAD for the chunk offset)
    uint32_t zero;            // 0; operand of the injected instructions of EXTRA > 0 (timing adversary)
    uint32_t one;             // 1; multiplier that keeps an add on the FMA pipe (ADDR = 2)
    uint32_t* counts;         // COUNT variant only: per-chunk read counters (inclusion experiment)
    uint64_t* cta_trace;      // optional: per CTA {smid, start ns, end ns, clock64 span} (diagnostics)
    uint32_t slice_shift;     // ADDR == 3 (cluster-distributed SMEM): log2 of the bytes each CTA holds
    uint64_t* progress;       // PROBE bit 5 only: per CTA, %globaltimer every progress_every trips
    uint32_t progress_every;  //   (progress[blockIdx.x * progress_slots + k]); diagnostics
    uint32_t progress_slots;
    // round 2 experiments
    uint64_t persist_bytes;   // LD 5/6: chunks below this byte offset are loaded with evict_last
    int64_t copy_delta;       // memory-copy adversary: picks are READ at dp + copy_delta (a clean
                              // copy elsewhere) while dp itself is folded (MEMCOPY knob)
};

// The region staged in shared memory (SMEM placement): namespace-scope so the
// round can address it with a constant base (LDS [v + const]).
extern __shared__ __align__(128) uint32_t smem_words[];

// R1 state step with a selectable lowering of each 64-bit shift-xor.
// XS bit k set => step k uses IMAD.WIDE.U32 by 2^s on the FMA pipe to
// produce both 32-bit halves of the cross-word shift, instead of the funnel
// shift on the ALU pipe.  Same function either way (xorshift64 (12,25,27)).
template <int XS>
__device__ __forceinline__ void xorshift_split(uint32_t& lo, uint32_t& hi, const KernelArgs& args) {
    // x ^= x >> 12
    if constexpr (XS & 8) {
        lo = lo ^ __funnelshift_r(lo, hi, 12);
        hi = hi ^ __umulhi(hi, args.p2[0]);                                // hi >> 12 on the FMA pipe
    } else if constexpr (XS & 1) {
        const uint64_t w = static_cast<uint64_t>(hi) * args.p2[0];         // {hi << 20, hi >> 12}
        lo = lo ^ (lo >> 12) ^ static_cast<uint32_t>(w);
        hi = hi ^ static_cast<uint32_t>(w >> 32);
    } else {
        lo = lo ^ __funnelshift_r(lo, hi, 12);
        hi = hi ^ (hi >> 12);
    }
    // x ^= x << 25
    if constexpr (XS & 2) {
        const uint64_t w = static_cast<uint64_t>(lo) * args.p2[1];         // {lo << 25, lo >> 7}
        hi = hi ^ (hi << 25) ^ static_cast<uint32_t>(w >> 32);
        lo = lo ^ static_cast<uint32_t>(w);
    } else {
        hi = hi ^ __funnelshift_l(lo, hi, 25);
        lo = lo ^ (lo << 25);
    }
    // x ^= x >> 27
    if constexpr (XS & 8) {
        lo = lo ^ __funnelshift_r(lo, hi, 27);
        hi = hi ^ __umulhi(hi, args.p2[2]);                                // hi >> 27 on the FMA pipe
    } else if constexpr (XS & 4) {
        const uint64_t w = static_cast<uint64_t>(hi) * args.p2[2];         // {hi << 5, hi >> 27}
        lo = lo ^ (lo >> 27) ^ static_cast<uint32_t>(w);
        hi = hi ^ static_cast<uint32_t>(w >> 32);
    } else {
        lo = lo ^ __funnelshift_r(lo, hi, 27);
        hi = hi ^ (hi >> 27);
    }
}

// One SCS-2 round (R1-R9) for this thread.
//   P        words per pick (1, 4, 8)
//   SMEM     region in shared memory (else read from global)
//   STRADDLE the region's chunk addresses may differ in their high 32 bits
//            (else hi32(dp) == hi32(base) for every chunk, host-checked)
//   XS       xorshift lowering (see xorshift_split)
//   EXTRA    number of result-neutral instructions injected (when `inject`) into
//            the round (0 in the product; > 0 only for the timing-adversary
//            experiment, the B200 analogue of Table 1 Exp 2's
//            "adversarial NOP"; the kernel injects them every EVERY
//            rounds of the unrolled trip, or in its first round when EVERY = 0)
//   COUNT    also count reads per chunk into args.counts (the memory-region
//            inclusion experiment); not in the timed path
// SCS-2 R6 / R9 odd multipliers: round index, high DP word, exchanged value.
constexpr uint32_t kKR = 0x9E3779B1u, kKH = 0x85EBCA77u, kKX = 0xC2B2AE3Du;

template <int P, bool SMEM, bool STRADDLE, int XS, int ADDR = 0, int LD = 0, int EXTRA = 0, bool COUNT = false,
          int PROBE = 0, int MEMCOPY = 0, int BAL = 0>
__device__ __forceinline__ void scs_round(uint32_t (&a)[kAccum], uint32_t& xlo, uint32_t& xhi, uint32_t r,
                                           uint64_t base, uint32_t nc_mask, uint32_t src_lane,
                                           const KernelArgs& args, uint64_t policy = 0, bool inject = false,
                                           uint64_t policy_lo = 0) {
    // R1
    xorshift_split<XS>(xlo, xhi, args);
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
    // R4, R5, R6 (first part)
    Pick<P> d;
    uint32_t t;
    if constexpr (SMEM && !STRADDLE && ADDR == 3) {
        // region distributed over the cluster's shared memories: CTA rank k holds
        // bytes [k << slice_shift, (k+1) << slice_shift); read through DSMEM
        const uint32_t v = i * args.four_p;
        const uint32_t owner = v >> args.slice_shift;
        const uint32_t local = smem_u32(smem_words) + (v & ((1u << args.slice_shift) - 1u));
        uint32_t raddr;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(local), "r"(owner));
        if constexpr (P == 1) {
            asm volatile("ld.shared::cluster.b32 %0, [%1];" : "=r"(d.w[0]) : "r"(raddr) : "memory");
        } else {
#pragma unroll
            for (int h = 0; h < P / 4; ++h)
                asm volatile("ld.shared::cluster.v4.b32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(d.w[4 * h]), "=r"(d.w[4 * h + 1]), "=r"(d.w[4 * h + 2]), "=r"(d.w[4 * h + 3])
                             : "r"(raddr + 16 * h) : "memory");
        }
        t = static_cast<uint32_t>(y) + (r * kKR + static_cast<uint32_t>(base) + static_cast<uint32_t>(base >> 32) * kKH) + v;
    } else if constexpr (SMEM && !STRADDLE && ADDR == 4) {
        // as ADDR == 2, with the whole warp-uniform bracket folded into the chunk-offset IMAD
        const uint32_t addr = i * args.four_p + smem_u32(smem_words);
        const uint32_t ur = r * kKR + static_cast<uint32_t>(base) + static_cast<uint32_t>(base >> 32) * kKH;
        if constexpr (PROBE & 1) d.w[0] = addr;                 // probe only: no shared-memory load
        else d = load_shared_addr<P>(addr);
        t = static_cast<uint32_t>(y) * args.one + (i * args.four_p + ur);
    } else if constexpr (SMEM && !STRADDLE && ADDR == 7) {
        // hybrid placement: the first region_bytes of the region are staged in shared
        // memory, the rest is read from global (L1/L2); each lane loads from whichever
        // holds its chunk (predicated LDS / LDG, so a lane touches one of the two)
        const uint32_t v = i * args.four_p;
        const uint32_t saddr = v + smem_u32(smem_words);
        const uint64_t gaddr = base + v;
        const uint32_t staged = args.region_bytes;
        if constexpr (P == 1) {
            asm volatile("{\n\t.reg .pred p;\n\t"
                         "setp.lt.u32 p, %1, %2;\n\t"
                         "@p ld.shared.b32 %0, [%3];\n\t"
                         "@!p ld.global.nc.b32 %0, [%4];\n\t}"
                         : "=r"(d.w[0]) : "r"(v), "r"(staged), "r"(saddr), "l"(gaddr));
        } else if constexpr (P == 4) {
            asm volatile("{\n\t.reg .pred p;\n\t"
                         "setp.lt.u32 p, %4, %5;\n\t"
                         "@p ld.shared.v4.b32 {%0,%1,%2,%3}, [%6];\n\t"
                         "@!p ld.global.nc.v4.b32 {%0,%1,%2,%3}, [%7];\n\t}"
                         : "=r"(d.w[0]), "=r"(d.w[1]), "=r"(d.w[2]), "=r"(d.w[3])
                         : "r"(v), "r"(staged), "r"(saddr), "l"(gaddr));
        } else {
            asm volatile("{\n\t.reg .pred p;\n\t"
                         "setp.lt.u32 p, %8, %9;\n\t"
                         "@p ld.shared.v4.b32 {%0,%1,%2,%3}, [%10];\n\t"
                         "@p ld.shared.v4.b32 {%4,%5,%6,%7}, [%10+16];\n\t"
                         "@!p ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%11];\n\t}"
                         : "=r"(d.w[0]), "=r"(d.w[1]), "=r"(d.w[2]), "=r"(d.w[3]),
                           "=r"(d.w[4]), "=r"(d.w[5]), "=r"(d.w[6]), "=r"(d.w[7])
                         : "r"(v), "r"(staged), "r"(saddr), "l"(gaddr));
        }
        t = static_cast<uint32_t>(y) + (r * kKR + static_cast<uint32_t>(base) + static_cast<uint32_t>(base >> 32) * kKH) + v;
    } else if constexpr (SMEM && !STRADDLE && ADDR == 8) {
        // hybrid placement as ADDR == 7 with the address arithmetic on the FMA pipe:
        // shared address and 64-bit global address as IMAD / IMAD.WIDE, and the R6
        // bracket folded as in ADDR == 4
        const uint32_t saddr = i * args.four_p + smem_u32(smem_words);
        const uint64_t gaddr = static_cast<uint64_t>(i) * args.four_p + (MEMCOPY ? base + args.copy_delta : base);
        const uint32_t staged_chunks = args.region_bytes / args.four_p;   // loop-invariant
        const uint32_t ur = r * kKR + static_cast<uint32_t>(base) + static_cast<uint32_t>(base >> 32) * kKH;
        static_assert(P == 1 || LD == 0, "ADDR 8 cache-operator variants are P = 1 forms");
        if constexpr (LD == 5 || LD == 6) {
            // round 2: keep a fixed window of the in-place part in L1 -- chunks in
            // [staged, staged + persist_bytes) load with .L1::evict_last, the rest with
            // .L1::no_allocate (LD 5) or .L1::evict_first (LD 6)
            const uint32_t win = static_cast<uint32_t>(args.persist_bytes) / args.four_p + staged_chunks;
            if constexpr (LD == 5)
                asm volatile("{\n\t.reg .pred ps, pw, pn;\n\t"
                             "setp.lt.u32 ps, %1, %2;\n\t"
                             "setp.lt.u32 pw, %1, %5;\n\t"
                             "setp.ge.and.u32 pn, %1, %2, pw;\n\t"
                             "@ps ld.shared.b32 %0, [%3];\n\t"
                             "@pn ld.global.nc.L1::evict_last.b32 %0, [%4];\n\t"
                             "@!pw ld.global.nc.L1::no_allocate.b32 %0, [%4];\n\t}"
                             : "=r"(d.w[0]) : "r"(i), "r"(staged_chunks), "r"(saddr), "l"(gaddr), "r"(win));
            else
                asm volatile("{\n\t.reg .pred ps, pw, pn;\n\t"
                             "setp.lt.u32 ps, %1, %2;\n\t"
                             "setp.lt.u32 pw, %1, %5;\n\t"
                             "setp.ge.and.u32 pn, %1, %2, pw;\n\t"
                             "@ps ld.shared.b32 %0, [%3];\n\t"
                             "@pn ld.global.nc.L1::evict_last.b32 %0, [%4];\n\t"
                             "@!pw ld.global.nc.L1::evict_first.b32 %0, [%4];\n\t}"
                             : "=r"(d.w[0]) : "r"(i), "r"(staged_chunks), "r"(saddr), "l"(gaddr), "r"(win));
        } else if constexpr (LD == 1)        // round 2: global part without L1 allocation
            asm volatile("{\n\t.reg .pred p;\n\t"
                         "setp.lt.u32 p, %1, %2;\n\t"
                         "@p ld.shared.b32 %0, [%3];\n\t"
                         "@!p ld.global.nc.L1::no_allocate.b32 %0, [%4];\n\t}"
                         : "=r"(d.w[0]) : "r"(i), "r"(staged_chunks), "r"(saddr), "l"(gaddr));
        else if constexpr (LD == 2)   // round 2: global part cached at L2 only
            asm volatile("{\n\t.reg .pred p;\n\t"
                         "setp.lt.u32 p, %1, %2;\n\t"
                         "@p ld.shared.b32 %0, [%3];\n\t"
                         "@!p ld.global.cg.b32 %0, [%4];\n\t}"
                         : "=r"(d.w[0]) : "r"(i), "r"(staged_chunks), "r"(saddr), "l"(gaddr));
        else if constexpr (P == 1)
        asm volatile("{\n\t.reg .pred p;\n\t"
                     "setp.lt.u32 p, %1, %2;\n\t"
                     "@p ld.shared.b32 %0, [%3];\n\t"
                     "@!p ld.global.nc.b32 %0, [%4];\n\t}"
                     : "=r"(d.w[0]) : "r"(i), "r"(staged_chunks), "r"(saddr), "l"(gaddr));
        else if constexpr (P == 4)    // the product's P = 4 SAGE_HYBRID form (= ADDR 10, session 2)
            asm volatile("{\n\t.reg .pred p;\n\t"
                         "setp.lt.u32 p, %4, %5;\n\t"
                         "@p ld.shared.v4.b32 {%0,%1,%2,%3}, [%6];\n\t"
                         "@!p ld.global.nc.v4.b32 {%0,%1,%2,%3}, [%7];\n\t}"
                         : "=r"(d.w[0]), "=r"(d.w[1]), "=r"(d.w[2]), "=r"(d.w[3])
                         : "r"(i), "r"(staged_chunks), "r"(saddr), "l"(gaddr));
        else
            asm volatile("{\n\t.reg .pred p;\n\t"
                         "setp.lt.u32 p, %8, %9;\n\t"
                         "@p ld.shared.v4.b32 {%0,%1,%2,%3}, [%10];\n\t"
                         "@p ld.shared.v4.b32 {%4,%5,%6,%7}, [%10+16];\n\t"
                         "@!p ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%11];\n\t}"
                         : "=r"(d.w[0]), "=r"(d.w[1]), "=r"(d.w[2]), "=r"(d.w[3]),
                           "=r"(d.w[4]), "=r"(d.w[5]), "=r"(d.w[6]), "=r"(d.w[7])
                         : "r"(i), "r"(staged_chunks), "r"(saddr), "l"(gaddr));
        t = static_cast<uint32_t>(y) * args.one + (i * args.four_p + ur);
    } else if constexpr (SMEM && !STRADDLE && ADDR == 11) {
        // round 2 (session 2): the P = 1 hybrid with a whole-line L1 prefetch ahead of
        // each global-side pick (LD 0: prefetch.global.L1 of the pick's 128-B line, then
        // the load; LD 1: prefetch only the line, load with .L1::evict_last), to test
        // whether line fills raise the L1 hit rate without costing L1->L2 requests
        static_assert(P == 1, "ADDR 11 is a P = 1 form");
        const uint32_t saddr = i * args.four_p + smem_u32(smem_words);
        const uint64_t gaddr = static_cast<uint64_t>(i) * args.four_p + base;
        const uint32_t staged_chunks = args.region_bytes / args.four_p;   // loop-invariant
        const uint32_t ur = r * kKR + static_cast<uint32_t>(base) + static_cast<uint32_t>(base >> 32) * kKH;
        if constexpr (LD == 1)
            asm volatile("{\n\t.reg .pred p;\n\t"
                         "setp.lt.u32 p, %1, %2;\n\t"
                         "@!p prefetch.global.L1 [%4];\n\t"
                         "@p ld.shared.b32 %0, [%3];\n\t"
                         "@!p ld.global.nc.L1::evict_last.b32 %0, [%4];\n\t}"
                         : "=r"(d.w[0]) : "r"(i), "r"(staged_chunks), "r"(saddr), "l"(gaddr));
        else
            asm volatile("{\n\t.reg .pred p;\n\t"
                         "setp.lt.u32 p, %1, %2;\n\t"
                         "@!p prefetch.global.L1 [%4];\n\t"
                         "@p ld.shared.b32 %0, [%3];\n\t"
                         "@!p ld.global.nc.b32 %0, [%4];\n\t}"
                         : "=r"(d.w[0]) : "r"(i), "r"(staged_chunks), "r"(saddr), "l"(gaddr));
        t = static_cast<uint32_t>(y) * args.one + (i * args.four_p + ur);
    } else if constexpr (SMEM && !STRADDLE && ADDR == 10) {
        // round 2: the ADDR 8 hybrid (FMA-pipe addressing, R6 bracket folded into the
        // chunk-offset IMAD) for P = 4 / 8: LDS.128 x P/4 from the staged prefix, one
        // 128 / 256-bit LDG from global
        static_assert(P == 4 || P == 8, "ADDR 10 is the P = 4 / 8 hybrid form");
        const uint32_t saddr = i * args.four_p + smem_u32(smem_words);
        const uint64_t gaddr = static_cast<uint64_t>(i) * args.four_p + base;
        const uint32_t staged_chunks = args.region_bytes / args.four_p;   // loop-invariant
        const uint32_t ur = r * kKR + static_cast<uint32_t>(base) + static_cast<uint32_t>(base >> 32) * kKH;
        if constexpr (P == 4) {
            asm volatile("{\n\t.reg .pred p;\n\t"
                         "setp.lt.u32 p, %4, %5;\n\t"
                         "@p ld.shared.v4.b32 {%0,%1,%2,%3}, [%6];\n\t"
                         "@!p ld.global.nc.v4.b32 {%0,%1,%2,%3}, [%7];\n\t}"
                         : "=r"(d.w[0]), "=r"(d.w[1]), "=r"(d.w[2]), "=r"(d.w[3])
                         : "r"(i), "r"(staged_chunks), "r"(saddr), "l"(gaddr));
        } else {
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
    } else if constexpr (SMEM && !STRADDLE && ADDR == 9) {
        // round 2: hybrid over a 2-CTA cluster.  CTA rank k stages bytes [k*S, (k+1)*S) of
        // the region (S = region_bytes); a pick below 2S is read from the owner's shared
        // memory (local LDS, or DSMEM from the partner CTA), the rest from global (L1/L2)
        static_assert(P == 1, "ADDR 9 is a P = 1 form");
        uint32_t crank;
        asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
        const uint32_t v = i * args.four_p;
        const uint32_t S = args.region_bytes;
        const uint32_t owner = v >= S ? 1u : 0u;
        const uint32_t saddr = v - owner * S + smem_u32(smem_words);
        const uint64_t gaddr = static_cast<uint64_t>(i) * args.four_p + base;
        const uint32_t ur = r * kKR + static_cast<uint32_t>(base) + static_cast<uint32_t>(base >> 32) * kKH;
        uint32_t raddr;
        asm("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(saddr), "r"(owner));
        asm volatile("{\n\t.reg .pred pn, pl, pr;\n\t"
                     "setp.lt.u32 pn, %1, %2;\n\t"                 // staged in the cluster
                     "setp.eq.and.u32 pl, %3, %4, pn;\n\t"         // ... in this CTA
                     "setp.ne.and.u32 pr, %3, %4, pn;\n\t"         // ... in the partner CTA
                     "@!pn ld.global.nc.b32 %0, [%5];\n\t"
                     "@pl ld.shared.b32 %0, [%6];\n\t"
                     "@pr ld.shared::cluster.b32 %0, [%7];\n\t"
                     "}"
                     : "=r"(d.w[0]) : "r"(v), "r"(2u * S), "r"(owner), "r"(crank), "l"(gaddr), "r"(saddr), "r"(raddr)
                     : "memory");
        t = static_cast<uint32_t>(y) * args.one + (i * args.four_p + ur);
    } else if constexpr (SMEM && !STRADDLE && ADDR == 5) {
        // lo32(y) + 4P*i in one IMAD, then the warp-uniform bracket
        const uint32_t addr = i * args.four_p + smem_u32(smem_words);
        const uint32_t ur = r * kKR + static_cast<uint32_t>(base) + static_cast<uint32_t>(base >> 32) * kKH;
        d = load_shared_addr<P>(addr);
        t = (i * args.four_p + static_cast<uint32_t>(y)) + ur;
    } else if constexpr (SMEM && !STRADDLE && ADDR == 6) {
        // lo32(y)*1 + addr (FMA pipe), then the warp-uniform bracket (which absorbs -smem)
        const uint32_t addr = i * args.four_p + smem_u32(smem_words);
        const uint32_t ur = r * kKR + (static_cast<uint32_t>(base) - smem_u32(smem_words)) +
                            static_cast<uint32_t>(base >> 32) * kKH;
        d = load_shared_addr<P>(addr);
        t = (static_cast<uint32_t>(y) * args.one + addr) + ur;
    } else if constexpr (SMEM && !STRADDLE && ADDR == 2) {
        // both chunk offsets and the R6 add as IMADs (FMA pipe), sparing the ALU pipe
        const uint32_t addr = i * args.four_p + smem_u32(smem_words);
        const uint32_t lo_dp = i * args.four_p + static_cast<uint32_t>(base);
        d = load_shared_addr<P>(addr);
        t = static_cast<uint32_t>(y) * args.one + lo_dp + (r * kKR + static_cast<uint32_t>(base >> 32) * kKH);
    } else if constexpr (SMEM && !STRADDLE && ADDR == 1) {
        // shared-window address of the chunk on the FMA pipe; lo32(dp) = addr + (lo32(base) - smem)
        const uint32_t addr = i * args.four_p + smem_u32(smem_words);
        d = load_shared_addr<P>(addr);
        const uint32_t base_minus_smem = static_cast<uint32_t>(base) - smem_u32(smem_words);   // loop-invariant
        // lo32(y) + r*KR + lo32(dp) + hi32(dp)*KH with lo32(dp) = addr + base_minus_smem; the bracket is
        // warp-uniform (uniform datapath)
        t = static_cast<uint32_t>(y) + (r * kKR + base_minus_smem + static_cast<uint32_t>(base >> 32) * kKH) + addr;
    } else if constexpr (SMEM && !STRADDLE) {
        const uint32_t v = i * (4u * P);                         // byte offset of the chunk
        d = load_shared<P>(smem_words + static_cast<size_t>(i) * P);
        t = static_cast<uint32_t>(y) + (r * kKR + static_cast<uint32_t>(base) + static_cast<uint32_t>(base >> 32) * kKH) + v;
    } else {
        const uint64_t dp = base + static_cast<uint64_t>(i) * (4u * P);   // R5 (= the global load address)
        if constexpr (SMEM) d = load_shared<P>(smem_words + static_cast<size_t>(i) * P);
        else if constexpr (MEMCOPY) d = load_global<P, LD>(reinterpret_cast<const uint32_t*>(dp + args.copy_delta), policy);
        else if constexpr (LD >= 5)
            d = load_global<P, LD>(reinterpret_cast<const uint32_t*>(dp),
                                   static_cast<uint64_t>(i) * (4u * P) < args.persist_bytes ? policy_lo : policy);
        else d = load_global<P, LD>(reinterpret_cast<const uint32_t*>(dp), policy);
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
        // BAL > 0 (round-2 prototype of a pipe-balanced round, NOT SCS-2): BAL extra
        // multiply-adds on the t chain, spread over R7 (t = t * odd + a[j ^ 8])
        if constexpr (BAL > 0) {
            if ((j + 1) % (kAccum / BAL) == 0 && (j + 1) / (kAccum / BAL) <= BAL)
                t = t * args.mul[(j + 5) & 15] + a[j ^ 8];
        }
    }
    // injected adversary work: dependent ALU ops that leave t unchanged (t ^ 0)
    if (inject) {
        // EXTRA > 0: dependent ALU-pipe ops (t ^ 0); EXTRA < 0: dependent FMA-pipe ops (t * 1)
#pragma unroll
        for (int e = 0; e < (EXTRA > 0 ? EXTRA : -EXTRA); ++e) {
            if constexpr (EXTRA > 0) t ^= args.zero;
            else t = t * args.one;
        }
    }
    // R8
    t = t + (t >> (C & 31u));
    // R9 (SCS-2: multiply-add exchange)
    if constexpr (PROBE & 2) a[kAccum - 1] = a[kAccum - 1] * kKX + t;    // probe only: no exchange
    else a[kAccum - 1] = a[kAccum - 1] * kKX + __shfl_sync(0xFFFFFFFFu, t, src_lane);
}

//   PROBE    measurement-only instruction-mix probes (never in the product; the
//            checksum is then not SCS-2): bit 0 replaces the pick's shared-memory
//            load by its address (ADDR == 4 only), bit 1 the neighbour exchange by
//            the lane's own t, so the loop keeps only its integer arithmetic;
//            bit 2 (result-neutral, ILP > 1) staggers the lane states: each state's
//            round starts with x += a'[0] * 0 (bit 3: a'[8]) on the other state's
//            accumulator, an FMA-pipe dependency that offsets the two chains;
//            bit 4 (result-neutral) emits the unrolled trip lane-state-major;
//            bit 5 (result-neutral) stamps a per-CTA progress trace (args.progress)
//   PAD      registers reserved (kept live across the round loop, unused) so that
//            an ILP > 1 kernel allocates the whole register file
//   SYNC     > 0: a CTA barrier every SYNC trips of the round loop (result-neutral;
//            bounds how far the warps of a CTA drift apart before the final reduction)
//   FEXTRA   timing adversary only (0 in the product): the adversary's own work
//            alongside the checksum, |FEXTRA| dependent ops per round per lane
//            state on a chain independent of the checksum state -- FFMA (FP32,
//            either FMA pipe) for FEXTRA > 0, IMAD (FMA-heavy pipe) for FEXTRA < 0;
//            folded into the result as (value & 0), so the checksum is unchanged
//   ILP      logical SCS-2 warps per hardware warp: 1 = one lane state per
//            thread, 2 CTAs x 1024 threads per SM at 32 registers; 2 = two
//            independent lane states per thread (interleaved by ptxas), one
//            CTA x 1024 threads per SM at 57-64 registers (64 allocated) -- the same register file
//            and logical grid, but all 32 warps of the SM progress together.
template <int P, bool SMEM, bool STRADDLE, int XS, int UNROLL, int ADDR = 0, int LD = 0, int EXTRA = 0,
          bool COUNT = false, int EVERY = 0, int ILP = 1, int PROBE = 0, int PAD = 0, int SYNC = 0, int FEXTRA = 0,
          int MEMCOPY = 0, int BAL = 0>
__global__ void __launch_bounds__(ILP <= 2 ? 1024 : 512, ILP == 1 ? 2 : 1) sage_checksum_kernel(const KernelArgs args) {
    __shared__ uint64_t red[32];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint64_t t_start_ns;
    __shared__ long long c_start;

    // a13: CTA start time (kept in shared memory, not in registers)
    if (threadIdx.x == 0) {
        t_start_ns = globaltimer();
        c_start = clock64();
    }

    // a2: stage the region into shared memory (SMEM placement).
    if constexpr (SMEM) {
        const uint32_t bytes = args.region_bytes;
        if ((bytes & 15u) == 0) {
            if (threadIdx.x == 0) mbar_init(&bar, 1);
            __syncthreads();
            if (threadIdx.x == 0) {
                mbar_expect_tx(&bar, bytes);
                uint32_t src0 = 0;                       // ADDR == 3: this CTA's slice of the region
                if constexpr (ADDR == 3 || ADDR == 9) {
                    uint32_t rank;
                    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
                    src0 = rank * bytes;
                }
                constexpr uint32_t kChunk = 32768;
                for (uint32_t off = 0; off < bytes; off += kChunk) {
                    const uint32_t n = (bytes - off < kChunk) ? (bytes - off) : kChunk;
                    bulk_g2s(reinterpret_cast<char*>(smem_words) + off,
                             reinterpret_cast<const char*>(args.region) + (MEMCOPY ? args.copy_delta : 0) + src0 + off,
                             n, &bar);
                }
            }
            mbar_wait(&bar, 0);
            if constexpr (ADDR == 3 || ADDR == 9) {      // every slice staged before any remote read
                asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
            }
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
    uint64_t policy = 0;
    if constexpr (LD == 4 || LD == 5) policy = evict_first_policy();
    if constexpr (LD == 6) policy = evict_normal_policy();
    uint64_t policy_lo = 0;
    if constexpr (LD >= 5) policy_lo = evict_last_policy();

    // a10: round loop, UNROLL rounds per trip + remainder
    uint32_t r = 0;
    const uint32_t main_end = rounds - rounds % UNROLL;
    uint32_t trips_to_sync = SYNC;
    float fadv[ILP];                                   // FEXTRA > 0: the adversary's FP32 chain
    uint32_t iadv[ILP];                                // FEXTRA < 0: the adversary's integer chain
#pragma unroll
    for (int s = 0; s < ILP; ++s) {
        fadv[s] = static_cast<float>(lane + s);
        iadv[s] = lane + s;
    }
    [[maybe_unused]] uint32_t trip = 0;
    for (; r < main_end; r += UNROLL) {
        if constexpr (PROBE & 32) {
            // progress trace (diagnostics, result-neutral): thread 0 stamps %globaltimer
            if (threadIdx.x == 0 && trip % args.progress_every == 0) {
                const uint32_t k = trip / args.progress_every;
                if (k < args.progress_slots) args.progress[static_cast<uint64_t>(blockIdx.x) * args.progress_slots + k] =
                    globaltimer();
            }
            ++trip;
        }
        if constexpr (SYNC > 0) {
            // keep the CTA's warps within SYNC trips of each other (result-neutral)
            if (--trips_to_sync == 0) {
                trips_to_sync = SYNC;
                __syncthreads();
            }
        }
#pragma unroll
        for (int uu = 0; uu < UNROLL * ILP; ++uu) {
            // source order of the unrolled trip: round-major (u, s) by default;
            // PROBE bit 4 (result-neutral) emits it lane-state-major (s, u) instead
            const int u = (PROBE & 16) ? uu % UNROLL : uu / ILP;
            const int s = (PROBE & 16) ? uu / UNROLL : uu % ILP;
            {
                if constexpr (ILP > 1 && (PROBE & 4)) {
                    // stagger: a result-neutral FMA-pipe dependency (x += a'[K] * 0) on a
                    // value the other lane state produces early in its last round
                    constexpr int kDep = (PROBE & 8) ? 8 : 0;
                    xlo[s] = a[(s + ILP - 1) % ILP][kDep] * args.zero + xlo[s];
                }
                scs_round<P, SMEM, STRADDLE, XS, ADDR, LD, EXTRA, COUNT, PROBE, MEMCOPY, BAL>(
                    a[s], xlo[s], xhi[s], r + u, base, nc_mask, src_lane, args, policy,
                    EVERY > 0 ? (u % EVERY == 0) : (u == 0), policy_lo);
#pragma unroll
                for (int e = 0; e < (FEXTRA > 0 ? FEXTRA : -FEXTRA); ++e) {
                    if constexpr (FEXTRA > 0) fadv[s] = fmaf(fadv[s], 1.0001f, 0.5f);
                    else iadv[s] = iadv[s] * args.mul[e & 15] + args.one;
                }
            }
        }
    }
    for (; r < rounds; ++r) {
#pragma unroll
        for (int s = 0; s < ILP; ++s)
            scs_round<P, SMEM, STRADDLE, XS, ADDR, LD, EXTRA, COUNT, PROBE, MEMCOPY, BAL>(a[s], xlo[s], xhi[s], r, base, nc_mask, src_lane,
                                                                      args, policy, true, policy_lo);
    }

    if constexpr (FEXTRA != 0) {
#pragma unroll
        for (int s = 0; s < ILP; ++s)          // keep the adversary's chain live: xlo ^= v & 0
            xlo[s] ^= (FEXTRA > 0 ? __float_as_uint(fadv[s]) : iadv[s]) & args.zero;
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
            if (args.cta_trace) {
                uint32_t smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                uint64_t* tr = args.cta_trace + 4ull * blockIdx.x;
                tr[0] = smid;
                tr[1] = t_start_ns;
                tr[2] = t_end_ns;
                tr[3] = static_cast<uint64_t>(c_end - c_start);
            }
        }
    }
    if constexpr (ADDR == 3 || ADDR == 9) {              // keep this CTA's slice alive for remote readers
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
}

// Host-side helper: fill the constant-bank tables of KernelArgs.
inline void fill_tables(KernelArgs& args, uint32_t P) {
    args.four_p = 4u * P;
    args.zero = 0;
    args.one = 1;
    for (int j = 0; j < kAccum; ++j) args.mul[j] = mul_of(j);
    args.p2[0] = 1u << 20;
    args.p2[1] = 1u << 25;
    args.p2[2] = 1u << 5;
}

}  // namespace sage_lab
