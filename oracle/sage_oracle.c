/*
 * sage_oracle.c -- plain CPU oracle for SCS-2, the SAGE self-checksumming
 * verification-function loop (arXiv 2209.03125).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2209_03125_b200/) never links, imports or calls it;
 * it shares no code, header, table or constant generator with the CUDA path.
 *
 * Citation keys: P:n = PAPER.md line n, S:n = SPEC.md line n.
 * The definition written out here is SCS-2: SURVEY.md
 * section 8(c)'s SCS-1 (readings Q1-Q20) with R6 and R9 combining by
 * multiply-add instead of XOR so the loop loads both integer pipes
 * (DESIGN.md "SCS-1 -> SCS-2").
 *
 * Deliberately plain: scalar uint32/uint64 arithmetic, one step per line in
 * the order the definition states, no intrinsics, no blocking, no fusion.
 * A warp (32 lanes) is the unit of work because R9 couples its lanes.
 *
 * Build: gcc -O2 -shared -fPIC -o liboracle.so sage_oracle.c
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>

#define WARP 32
#define K 16

/* xorshift64* multiplier, S:241 ("multiplier 2685821657736338717"). */
static const uint64_t M64 = 0x2545F4914F6CDD1DULL;
/* SplitMix64 golden-ratio increment (Steele, Lea, Flood 2014). */
static const uint64_t GAMMA = 0x9E3779B97F4A7C15ULL;

/* R7 tables (reading Q6): multiplier exponent L[j] (MUL = 2^L+1)
 * and rotate amount S[j] per accumulator j.  "alternating ... shifts with
 * addition ... arbitrarily chosen shift size". */
static const unsigned L_TAB[K] = {5, 11, 3, 17, 9, 23, 7, 13, 29, 2, 19, 6, 15, 27, 4, 21};
static const unsigned S_TAB[K] = {7, 13, 19, 3, 25, 9, 17, 5, 11, 29, 2, 23, 14, 6, 27, 18};
/* R6 / R9 odd multipliers (SCS-2): round index, high DP word, exchanged value. */
static const uint32_t KR = 0x9E3779B1u, KH = 0x85EBCA77u, KX = 0xC2B2AE3Du;

/* ---- helpers -------------------------------------------------------------- */

/* SplitMix64 finaliser sm(z) (Vigna, splitmix64.c). Used by I1 (Q3). */
uint64_t sage_oracle_splitmix_mix(uint64_t z)
{
    z = z ^ (z >> 30);
    z = z * 0xBF58476D1CE4E5B9ULL;
    z = z ^ (z >> 27);
    z = z * 0x94D049BB133111EBULL;
    z = z ^ (z >> 31);
    return z;
}

/* xorshift64 state step with the (12,25,27) triple. */
uint64_t sage_oracle_xs(uint64_t x)
{
    x = x ^ (x >> 12);
    x = x ^ (x << 25);
    x = x ^ (x >> 27);
    return x;
}

static uint32_t hi32(uint64_t v) { return (uint32_t)(v >> 32); }
static uint32_t lo32(uint64_t v) { return (uint32_t)(v & 0xFFFFFFFFULL); }

/* rotate a u32 left by s, 1 <= s <= 31 */
static uint32_t rotl32(uint32_t v, unsigned s) { return (v << s) | (v >> (32u - s)); }

/* little-endian u32 word k of the region (Q19) */
static uint32_t word_le(const uint8_t *region, uint64_t k)
{
    const uint8_t *b = region + 4 * k;
    return (uint32_t)b[0] | ((uint32_t)b[1] << 8) | ((uint32_t)b[2] << 16) | ((uint32_t)b[3] << 24);
}

/* ---- I1-I3: per-thread seeding ("uses its challenge as a seed value
 * to initialize all per-thread state with random data and a PRNG") ---------- */
void sage_oracle_thread_init(uint64_t nonce, uint64_t g, uint32_t a[K], uint64_t *x_out)
{
    /* I1: the (g+1)-th SplitMix64 output of the stream seeded with nonce */
    uint64_t s = sage_oracle_splitmix_mix(nonce + (g + 1) * GAMMA);
    /* I2: xorshift state must be non-zero */
    uint64_t x = (s != 0) ? s : GAMMA;
    /* I3: sixteen xorshift64* outputs, high halves */
    for (int j = 0; j < K; j++) {
        x = sage_oracle_xs(x);
        a[j] = hi32(x * M64);
    }
    *x_out = x;
}

/* ---- one round r for all 32 lanes of a warp (P:638-655 steps 1-5, north_star
 * neighbour exchange).  nc = number of P-word chunks (power of two). -------- */
static void warp_round(uint32_t a[WARP][K], uint64_t x[WARP], uint32_t r,
                       const uint8_t *region, uint64_t nc, uint64_t base, unsigned P,
                       uint32_t *counts)
{
    uint32_t t_lane[WARP];
    for (int l = 0; l < WARP; l++) {
        /* R1: PRNG step */
        x[l] = sage_oracle_xs(x[l]);
        uint64_t y = x[l] * M64;
        /* R2: C = current checksum word (P:646 symbol C; Q2) */
        uint32_t C = a[l][K - 1];
        /* R3: chunk index; 4*C % data_size with power-of-two size (Q1) */
        uint64_t i = (uint64_t)(hi32(y) ^ C) & (nc - 1);
        /* inclusion experiment: count the pick of chunk i */
        if (counts != NULL)
            counts[i] += 1;
        /* R4: pseudo-random read of P consecutive words */
        uint32_t d[8];
        for (unsigned q = 0; q < P; q++)
            d[q] = word_le(region, (uint64_t)P * i + q);
        /* R5: data pointer = device VA of the picked chunk (Q9) */
        uint64_t dp = base + 4ULL * P * i;
        /* R6: iteration index and DP folded in, then the data (Q19) */
        uint32_t t = lo32(y) + r * KR + lo32(dp) + hi32(dp) * KH;
        for (unsigned q = 0; q < P; q++)
            t = rotl32(t, 5) + d[q];
        /* R7: strongly-ordered multiply-add / rotate-add chain */
        for (int j = 0; j < K; j++) {
            uint32_t mul = (1u << L_TAB[j]) + 1u;
            a[l][j] = a[l][j] * mul + t;
            t = a[l][j] + rotl32(t, S_TAB[j]);
        }
        /* R8: self-modifying instruction semantics x += x >> N, N = C mod 32
         * */
        t = t + (t >> (C & 31u));
        t_lane[l] = t;
    }
    /* R9: neighbour exchange from a snapshot (north_star; Q13) */
    for (int l = 0; l < WARP; l++)
        a[l][K - 1] = a[l][K - 1] * KX + t_lane[(l + 1) % WARP];
}

/* F1-F2: per-thread fold (Q11) */
uint64_t sage_oracle_fold(const uint32_t a[K], uint64_t x)
{
    uint32_t e = 0, o = 0;
    for (int j = 0; j < K; j += 2) e ^= a[j];
    for (int j = 1; j < K; j += 2) o ^= a[j];
    uint64_t f = ((uint64_t)o << 32) | (uint64_t)e;
    return f ^ x;
}

/* Argument check shared by the entry points below. Returns 0 if valid. */
static int check_args(const uint8_t *region, uint64_t nbytes, uint64_t base, uint64_t rounds, unsigned P)
{
    if (P != 1 && P != 4 && P != 8) return -1;
    if (region == NULL || nbytes == 0) return -1;
    if (nbytes % (4ULL * P) != 0) return -1;
    uint64_t nc = nbytes / (4ULL * P);
    if ((nc & (nc - 1)) != 0 || nc > (1ULL << 32)) return -1;
    uint64_t align = (4ULL * P > 16) ? 4ULL * P : 16;
    if (base % align != 0) return -1;
    if (rounds > 0xFFFFFFFFULL) return -1;
    return 0;
}

/*
 * Run rounds [r_begin, r_end) on an explicit warp state (state injection for
 * tests).  a: 32*16 u32 row-major [lane][j]; x: 32 u64.  Returns 0 / -1.
 */
int sage_oracle_warp_rounds(uint32_t *a_flat, uint64_t *x, const uint8_t *region, uint64_t nbytes,
                            uint64_t base, uint64_t r_begin, uint64_t r_end, unsigned P)
{
    if (check_args(region, nbytes, base, r_end, P) != 0 || r_begin > r_end) return -1;
    uint64_t nc = nbytes / (4ULL * P);
    uint32_t (*a)[K] = (uint32_t (*)[K])a_flat;
    for (uint64_t r = r_begin; r < r_end; r++)
        warp_round(a, x, (uint32_t)r, region, nc, base, P, NULL);
    return 0;
}

/*
 * Sum mod 2^64 of the folded states of the 32 threads g = 32*w .. 32*w+31.
 * This is the warp-level partial of the epilog.
 */
static int warp_sum_counted(uint64_t nonce, const uint8_t *region, uint64_t nbytes, uint64_t base,
                            uint64_t rounds, uint64_t w, unsigned P, uint64_t *warp_sum, uint32_t *counts)
{
    if (check_args(region, nbytes, base, rounds, P) != 0 || warp_sum == NULL) return -1;
    uint32_t a[WARP][K];
    uint64_t x[WARP];
    for (int l = 0; l < WARP; l++)
        sage_oracle_thread_init(nonce, 32ULL * w + (uint64_t)l, a[l], &x[l]);
    uint64_t nc = nbytes / (4ULL * P);
    for (uint64_t r = 0; r < rounds; r++)
        warp_round(a, x, (uint32_t)r, region, nc, base, P, counts);
    uint64_t sum = 0;
    for (int l = 0; l < WARP; l++)
        sum += sage_oracle_fold(a[l], x[l]);
    *warp_sum = sum;
    return 0;
}

int sage_oracle_warp(uint64_t nonce, const uint8_t *region, uint64_t nbytes, uint64_t base,
                     uint64_t rounds, uint64_t w, unsigned P, uint64_t *warp_sum)
{
    return warp_sum_counted(nonce, region, nbytes, base, rounds, w, P, warp_sum, NULL);
}

/*
 * Inclusion experiment: as sage_oracle_attest, and also adds to
 * counts[k] (Nc u32, caller-zeroed) the number of times chunk k is picked.
 */
int sage_oracle_attest_counts(uint64_t nonce, const uint8_t *region, uint64_t nbytes, uint64_t base,
                              uint64_t rounds, uint64_t blocks, uint64_t threads, unsigned P,
                              uint64_t *checksum, uint32_t *counts)
{
    if (checksum == NULL || counts == NULL || threads == 0 || threads % WARP != 0 || blocks == 0) return -1;
    uint64_t nwarps = blocks * threads / WARP;
    uint64_t total = 0;
    for (uint64_t w = 0; w < nwarps; w++) {
        uint64_t s;
        if (warp_sum_counted(nonce, region, nbytes, base, rounds, w, P, &s, counts) != 0) return -1;
        total += s;
    }
    *checksum = total;
    return 0;
}

/*
 * Whole attestation result: n = blocks*threads threads (threads % 32 == 0);
 * checksum = sum over all threads of F(thread) mod 2^64.
 */
int sage_oracle_attest(uint64_t nonce, const uint8_t *region, uint64_t nbytes, uint64_t base,
                       uint64_t rounds, uint64_t blocks, uint64_t threads, unsigned P, uint64_t *checksum)
{
    if (checksum == NULL || threads == 0 || threads % WARP != 0 || blocks == 0) return -1;
    uint64_t nwarps = blocks * threads / WARP;
    uint64_t total = 0;
    for (uint64_t w = 0; w < nwarps; w++) {
        uint64_t s;
        if (sage_oracle_warp(nonce, region, nbytes, base, rounds, w, P, &s) != 0) return -1;
        total += s;
    }
    *checksum = total;
    return 0;
}
