// sage_hash.cuh -- h = SHA-256(r || code) on the GPU (SAGE Eq. (9), P:536-543;
// SURVEY 8(f) NEXT #3): the verification function's authenticity check of the
// user kernel located in device memory, with a verifier-provided random r.
//
// SHA-256 over one message is a serial chain of 64-round compressions, so one
// thread does the compression while a producer warp keeps it fed: it gathers
// the padded message r || code || 0x80 || 0* || len64 into shared memory 32
// blocks at a time (one block per lane), expands each block's message
// schedule and stores K[t] + W[t] (FIPS 180-4 6.2.2 steps 1 and 4 folded), so
// the compressor's round is only the a..h update.  Producer and consumer are
// double-buffered through named barriers.
#pragma once
#include <stdint.h>

namespace sage {

constexpr int kHashRMax = 128;          // bytes of r carried in the kernel parameters
constexpr int kHashChunk = 32;          // message blocks per producer chunk (one per lane)

struct HashArgs {
    const uint8_t* code;
    uint64_t code_len;
    uint8_t* out;                       // 32 bytes, big-endian H0..H7
    uint32_t r_len;
    uint8_t r[kHashRMax];
};

__device__ __constant__ uint32_t kSha256K[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

__device__ __forceinline__ uint32_t rotr32(uint32_t x, uint32_t n) { return __funnelshift_r(x, x, n); }

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
    asm volatile("bar.sync %0, %1;" :: "r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(uint32_t id, uint32_t n) {
    asm volatile("bar.arrive %0, %1;" :: "r"(id), "r"(n) : "memory");
}

// byte p of the padded message (FIPS 180-4 5.1.1)
__device__ __forceinline__ uint32_t hash_msg_byte(const HashArgs& a, uint64_t p, uint64_t len, uint64_t lenpos) {
    if (p < a.r_len) return a.r[p];
    if (p < len) return __ldg(a.code + (p - a.r_len));
    if (p == len) return 0x80u;
    if (p >= lenpos) return static_cast<uint32_t>(((len * 8) >> (8 * (7 - (p - lenpos)))) & 0xFFu);
    return 0u;
}

// One CTA of 64 threads: warp 0 lane 0 compresses, warp 1 produces.
__global__ void __launch_bounds__(64, 1) sage_sha256_kernel(const HashArgs args) {
    __shared__ uint32_t kw[2][kHashChunk][64];        // K[t] + W[t] per block, double-buffered (16 KiB)
    __shared__ __align__(16) uint8_t bytes[kHashChunk * 64];   // producer staging of one chunk's message bytes

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint64_t len = args.r_len + args.code_len;
    const uint64_t nblocks = (len + 9 + 63) / 64;
    const uint64_t lenpos = nblocks * 64 - 8;
    const uint64_t nchunks = (nblocks + kHashChunk - 1) / kHashChunk;
    constexpr uint32_t kFull0 = 1, kEmpty0 = 3;       // named barriers 1,2 (full) and 3,4 (empty)

    if (warp == 1) {
        for (uint64_t c = 0; c < nchunks; ++c) {
            const uint32_t buf = static_cast<uint32_t>(c & 1);
            if (c >= 2) named_bar_sync(kEmpty0 + buf, 64);       // consumer released this buffer
            const uint64_t p0 = c * kHashChunk * 64;
            const uint64_t q0 = p0 - args.r_len;                      // offset of the chunk inside code
            const bool fast = p0 >= args.r_len && p0 + kHashChunk * 64 <= len &&
                              ((reinterpret_cast<uintptr_t>(args.code) + q0) & 15u) == 0;
            if (fast) {   // whole chunk inside code, 16-B aligned: coalesced 128-bit loads
                const uint4* src = reinterpret_cast<const uint4*>(args.code + q0);
#pragma unroll
                for (uint32_t k = 0; k < kHashChunk * 64 / 16 / 32; ++k)
                    reinterpret_cast<uint4*>(bytes)[lane + 32 * k] = __ldg(src + lane + 32 * k);
            } else {      // boundary chunks: r / code / padding byte by byte
                for (uint32_t k = lane; k < kHashChunk * 64; k += 32)
                    bytes[k] = static_cast<uint8_t>(p0 + k < nblocks * 64 ? hash_msg_byte(args, p0 + k, len, lenpos) : 0u);
            }
            __syncwarp();
            // lane = block within the chunk: schedule W (FIPS 6.2.2 step 1) + K
            uint32_t w[16];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint4 v = reinterpret_cast<const uint4*>(bytes + lane * 64)[q];
                w[4 * q + 0] = __byte_perm(v.x, 0, 0x0123);                     // big-endian words
                w[4 * q + 1] = __byte_perm(v.y, 0, 0x0123);
                w[4 * q + 2] = __byte_perm(v.z, 0, 0x0123);
                w[4 * q + 3] = __byte_perm(v.w, 0, 0x0123);
            }
#pragma unroll
            for (int t = 0; t < 16; ++t) kw[buf][lane][t] = w[t] + kSha256K[t];
#pragma unroll
            for (int t = 16; t < 64; ++t) {
                const uint32_t w15 = w[(t - 15) & 15], w2 = w[(t - 2) & 15];
                const uint32_t s0 = rotr32(w15, 7) ^ rotr32(w15, 18) ^ (w15 >> 3);
                const uint32_t s1 = rotr32(w2, 17) ^ rotr32(w2, 19) ^ (w2 >> 10);
                w[t & 15] = s1 + w[(t - 7) & 15] + s0 + w[t & 15];
                kw[buf][lane][t] = w[t & 15] + kSha256K[t];
            }
            __syncwarp();
            named_bar_arrive(kFull0 + buf, 64);
        }
    } else {
        uint32_t H[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
        for (uint64_t c = 0; c < nchunks; ++c) {
            const uint32_t buf = static_cast<uint32_t>(c & 1);
            named_bar_sync(kFull0 + buf, 64);
            if (lane == 0) {
                const uint64_t nb = (nblocks - c * kHashChunk < kHashChunk) ? nblocks - c * kHashChunk : kHashChunk;
                for (uint32_t b = 0; b < nb; ++b) {
                    uint32_t A = H[0], B = H[1], C = H[2], D = H[3], E = H[4], F = H[5], G = H[6], Hh = H[7];
                    const uint32_t* k = kw[buf][b];
#pragma unroll
                    for (int t = 0; t < 64; ++t) {
                        // T1 = h + S1(e) + Ch(e,f,g) + K[t] + W[t]; T2 = S0(a) + Maj(a,b,c)
                        // (FIPS 6.2.2 step 3), summed so that only S1 -> one add is on
                        // the e-chain: e' = S1 + (Ch + h + KW + d), a' = S1 + (Ch + h + KW) + T2
                        const uint32_t hk = Hh + k[t];
                        const uint32_t ch = (E & F) ^ (~E & G);
                        const uint32_t chhk = ch + hk;
                        const uint32_t chhkd = chhk + D;
                        const uint32_t S1 = rotr32(E, 6) ^ rotr32(E, 11) ^ rotr32(E, 25);
                        const uint32_t S0 = rotr32(A, 2) ^ rotr32(A, 13) ^ rotr32(A, 22);
                        const uint32_t maj = (A & B) ^ (A & C) ^ (B & C);
                        const uint32_t t2 = S0 + maj;
                        Hh = G; G = F; F = E; E = S1 + chhkd;
                        D = C; C = B; B = A; A = S1 + chhk + t2;
                    }
                    H[0] += A; H[1] += B; H[2] += C; H[3] += D; H[4] += E; H[5] += F; H[6] += G; H[7] += Hh;
                }
            }
            __syncwarp();
            if (c + 2 < nchunks) named_bar_arrive(kEmpty0 + buf, 64);
        }
        if (lane == 0) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                args.out[4 * i] = static_cast<uint8_t>(H[i] >> 24);
                args.out[4 * i + 1] = static_cast<uint8_t>(H[i] >> 16);
                args.out[4 * i + 2] = static_cast<uint8_t>(H[i] >> 8);
                args.out[4 * i + 3] = static_cast<uint8_t>(H[i]);
            }
        }
    }
}

}  // namespace sage
