/*
 * sage.h -- C ABI of the B200-native SAGE checksum hot path (libsage.so).
 *
 * The operation is the self-verifying checksum function of SAGE
 * (arXiv 2209.03125, section 5.2.2; loop steps at
 * lines 634-657): every resident thread is seeded from the verifier's challenge
 * (P:383-389), runs `rounds` iterations that read a pseudo-randomly chosen piece
 * of the checksummed region and fold it, the data pointer and the round index
 * into an ordered integer state, and the per-thread states are
 * summed warp -> block -> grid into one value.  The exact
 * arithmetic is SCS-2.
 *
 * Conventions for every function:
 *   - returns SAGE_OK (0) or a negative SAGE_E* code; never throws/aborts;
 *   - output structs are written only on success;
 *   - a wrong checksum is not an error: comparing against the expected value
 *     is the verifier's job;
 *   - sage_last_error() returns a thread-local detail string for the last failure;
 *   - every DEVICE buffer argument (region, per_warp_out, raw_out, counts_out,
 *     code) is checked with cudaPointerGetAttributes: host memory without a
 *     device mapping, or another device's allocation, is SAGE_EINVAL rather than
 *     a fault inside the kernel (managed and mapped pinned memory are accepted;
 *     the extent of the buffer cannot be checked and is the caller's contract).
 *
 * Ownership: the caller owns `region` (a device pointer, or a host pointer for
 * sage_attest_host) and must keep it alive and unmodified until the call
 * returns (for sage_attest_async: until the stream work completes).  The
 * result depends on the region's DEVICE virtual address because the data
 * pointer is folded in every round.  The context owns its result
 * buffers, its staging buffer for host regions and, when the config's stream is
 * NULL, its stream.
 *
 * Threads: every function may be called from any thread; calls on the same
 * context are serialised by a per-context lock (use one context per thread or
 * stream for concurrency).  The launch-count read is unsynchronised.
 *
 * Device: every function makes the context's device current for the call and
 * restores the caller's current device before returning.
 *
 * Stream ordering: work is enqueued on the config's stream, or -- stream NULL --
 * on a context-owned BLOCKING stream (cudaStreamDefault flags), which is ordered
 * with the legacy default stream: device buffers written on the legacy default
 * stream (plain CUDA calls, torch's default stream) before a call are complete
 * when the kernel reads them.  With a caller-supplied stream the caller orders its
 * own work (e.g. zeroes raw_out on that stream, see sage_attest_async).
 */
#ifndef SAGE_H
#define SAGE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SAGE_OK            0
#define SAGE_EINVAL       -1  /* bad argument (see each function) */
#define SAGE_EUNSUPPORTED -2  /* valid but not supported here (e.g. forced SMEM too large) */
#define SAGE_ENOMEM       -3  /* device or pinned host allocation failed */
#define SAGE_ECUDA        -4  /* CUDA runtime error; detail in sage_last_error() */

/* region placement */
#define SAGE_AUTO   0u  /* SMEM up to smem_region_max (64 KiB, or 128 KiB at the ILP-2 geometry:
                           P = 1, 1024-thread blocks, even block count); then HYBRID up to
                           1 MiB at that geometry (P = 4: HYBRID from 256 KiB to 1 MiB at
                           the same block geometry); else GLOBAL (always for P = 8) */
#define SAGE_SMEM   1u  /* region staged once per CTA into shared memory (TMA bulk copy) */
#define SAGE_GLOBAL 2u  /* region read in place from L2/HBM every round */
#define SAGE_HYBRID 3u  /* first min(region, 192 KiB) staged in shared memory, the rest read
                           in place; each pick loads from whichever holds it.  Needs P = 1
                           or 4, 1024-thread blocks, an even block count and a region whose chunk
                           addresses share their high 32 bits (one CTA x 1024 threads x 2
                           lane states per SM); SAGE_AUTO picks it for 128 KiB < region <=
                           1 MiB (P = 1) or 256 KiB <= region <= 1 MiB (P = 4) when those
                           hold */

typedef struct sage_ctx sage_ctx;

typedef struct {
    int      device;      /* CUDA device ordinal */
    uint32_t blocks;      /* grid size; 0 => 2 * SM count (full occupancy) */
    uint32_t threads;     /* block size, multiple of 32, <= 1024; 0 => 1024 */
    uint32_t pick_words;  /* P, words read per round: 1, 4 or 8; 0 => 1 */
    uint32_t placement;   /* SAGE_AUTO | SAGE_SMEM | SAGE_GLOBAL | SAGE_HYBRID */
    void*    stream;      /* cudaStream_t to launch on (borrowed); NULL => ctx-owned stream */
} sage_config;

typedef struct {
    uint64_t checksum;    /* sum over all threads of the folded state, mod 2^64 */
    uint64_t cycles;      /* max over CTAs of the CTA's clock64 duration */
    uint64_t elapsed_ns;  /* host CLOCK_MONOTONIC from before launch to result on host (t1 - t0) */
    uint64_t device_ns;   /* %globaltimer: last CTA end - first CTA start */
    uint64_t region_va;   /* device VA the region was read from (the `base` of SCS-2) */
    uint32_t placement;   /* SAGE_SMEM, SAGE_GLOBAL or SAGE_HYBRID actually used */
    uint32_t blocks;      /* logical grid (blocks x threads logical threads; see ilp) */
    uint32_t threads;     /* block size actually launched */
    uint32_t pick_words;  /* P actually used */
    uint32_t ilp;         /* logical lane states per hardware thread (1 or 2): the launch was
                             blocks/ilp CTAs of `threads`, covering the same blocks*threads
                             logical threads (the c2a kernel uses 2) */
    uint32_t tuned;       /* 1 if the kernel ran from sage_kernel_tuned.cubin (the c2a kernel with
                             control-bit-tuned scheduling hints, same instructions, DESIGN.md
                             section 8); 0 for the kernel embedded in the library */
} sage_result;

typedef struct {
    int      device;
    uint32_t sm_count;         /* cudaDevAttrMultiProcessorCount */
    uint32_t blocks, threads, pick_words, placement;
    uint32_t ctas_per_sm_smem; /* resident CTAs/SM of the SMEM kernel with a 64 KiB region */
    uint32_t ctas_per_sm_global;
    uint32_t regs_per_thread;  /* of the P-specific SMEM kernel, as compiled (allocated per warp in
                                  units of 256, i.e. rounded up to a multiple of 8 per thread) */
    uint64_t smem_region_max;  /* largest region (bytes) SAGE_AUTO stages into SMEM: 64 KiB,
                                  128 KiB at the ILP-2 geometry (see SAGE_AUTO) */
    uint32_t ilp_smem;         /* lane states per thread of that SMEM kernel (1 or 2) */
} sage_info;

/* Initialise the verification function on cfg->device ("Initialization of the
 * VF": the GPU allocates the VF's buffers before the verifier starts
 * challenging it).  The default grid occupies every SM with all its threads and
 * registers, 2 x SMs x 1024 threads, the B200 analogue of the A100's
 * 2 x 108 x 1024.  cfg may be NULL
 * (all defaults).  Allocates the 32-byte device result and its pinned host copy,
 * creates the stream if cfg->stream is NULL, and sets the dynamic shared-memory
 * limits of the kernels the context can stage into (the only kernel-attribute
 * change the library makes).  *out is owned by the caller; free it with
 * sage_checksum_destroy.
 * SAGE_EINVAL: threads % 32 != 0 or > 1024, pick_words not in {1,4,8},
 *              placement unknown, device ordinal out of range, out NULL.
 * SAGE_ENOMEM / SAGE_ECUDA: allocation or runtime failure (nothing is leaked). */
int sage_checksum_init(const sage_config* cfg, sage_ctx** out);

/* One attestation, synchronous (the verifier's challenge -> checksum exchange,
 * P:313-316; the checksum function P:369-463 with the loop of P:638-655 as
 * SCS-2, base = region).  The host time from before the
 * launch to the result on the host is out->elapsed_ns, the verifier's t1 - t0
 * (P:501).
 * region: DEVICE pointer (borrowed, read-only, must stay unmodified until the
 * call returns); region_bytes = 4 * P * Nc with Nc a power of two (<= 2^32);
 * region 16-byte aligned (32-byte for P = 8); rounds < 2^32 (R = 0 is allowed:
 * the seeded state is folded directly).  Returns when the result is on the host.
 * SAGE_EINVAL on a violated precondition or NULL pointer;
 * SAGE_EUNSUPPORTED when SAGE_SMEM was forced and the region does not fit, or
 * SAGE_HYBRID was forced without its geometry (see SAGE_HYBRID). */
int sage_attest(sage_ctx* ctx, uint64_t nonce, const void* region, size_t region_bytes,
                uint64_t rounds, sage_result* out);

/* As sage_attest, and also writes the per-warp partial sums of the epilog's
 * pairwise sum: n/32 u64 to per_warp_out (DEVICE pointer, may be
 * NULL; warp w = logical threads 32w..32w+31), so large configs can be checked on
 * sampled warps: sum of partials == checksum (mod 2^64). */
int sage_attest_debug(sage_ctx* ctx, uint64_t nonce, const void* region, size_t region_bytes,
                      uint64_t rounds, uint64_t* per_warp_out, sage_result* out);

/* Asynchronous form of sage_attest (same operation):
 * validates, then enqueues the checksum kernel on the context's stream and returns.  raw_out is a DEVICE buffer of 4 u64 that the
 * kernel accumulates into and that the CALLER must zero (on the same stream)
 * before the launch:
 *   raw_out[0] checksum, [1] max CTA cycles, [2] ~(first CTA start ns),
 *   [3] last CTA end ns.  per_warp_out may be NULL.  Decode with
 *   sage_decode_raw.  Safe to capture in a CUDA graph. */
int sage_attest_async(sage_ctx* ctx, uint64_t nonce, const void* region, size_t region_bytes,
                      uint64_t rounds, uint64_t* raw_out, uint64_t* per_warp_out);

/* Inclusion experiment (SAGE section 7.3): as sage_attest with GLOBAL placement,
 * and also counts how often each chunk is read.  counts_out: DEVICE buffer of
 * Nc = region_bytes / (4 * P) u32, zeroed by the call.  The checksum is the
 * same as sage_attest's for the same inputs; the timing is not representative
 * (one global atomic per pick). */
int sage_attest_coverage(sage_ctx* ctx, uint64_t nonce, const void* region, size_t region_bytes,
                         uint64_t rounds, uint32_t* counts_out, sage_result* out);

/* User-kernel authenticity check, SAGE Eq. (9): h = SHA-256(r || code)
 * computed on the GPU over `code_len` bytes of DEVICE memory at `code` (the user
 * kernel as located on the device) prefixed with the verifier's random value r
 * (HOST pointer, r_len <= 128 bytes; SPEC S:367 uses 32).  Synchronous; writes
 * the 32-byte big-endian digest to h_out (host) and, if non-NULL, the host wall
 * time of the call to *elapsed_ns.  SAGE_EINVAL: r_len > 128, NULL h_out, NULL
 * r or code with a non-zero length. */
int sage_kernel_hash(sage_ctx* ctx, const uint8_t* r, size_t r_len, const void* code, size_t code_len,
                     uint8_t* h_out, uint64_t* elapsed_ns);

/* Decode a raw 4 x u64 result (host copy of sage_attest_async's raw_out) into
 * checksum / cycles / device_ns (P:501 timing fields); SAGE_EINVAL on NULL. */
int sage_decode_raw(const uint64_t raw[4], sage_result* out);

/* End-to-end form of sage_attest over a HOST region (P:313-316 with the region
 * supplied by the host): copies the region host->device into a context-owned
 * device buffer (whose VA is reported in out->region_va and is the SCS-2 base),
 * attests, copies the 32-byte result back.  elapsed_ns covers the copies.
 * Pinned host memory gives the fastest copy.  region_bytes and rounds are
 * validated BEFORE the staging buffer is (re)allocated, so an invalid call
 * (SAGE_EINVAL) leaves the buffer and its VA unchanged; a larger valid region
 * reallocates it (new VA). */
int sage_attest_host(sage_ctx* ctx, uint64_t nonce, const void* host_region, size_t region_bytes,
                     uint64_t rounds, sage_result* out);

/* Device VA of the context-owned staging buffer sage_attest_host would use
 * for a region of region_bytes (allocating it if needed), so a verifier can
 * precompute the expected checksum ahead of time (the result depends
 * on the data pointer).  SAGE_EINVAL for an invalid region_bytes. */
int sage_host_region_va(sage_ctx* ctx, size_t region_bytes, uint64_t* va_out);

/* Placement the context would choose for region_bytes (SAGE_SMEM/SAGE_GLOBAL/SAGE_HYBRID;
 * a HYBRID region whose chunk addresses straddle a 4 GiB boundary runs GLOBAL). */
int sage_placement_for(sage_ctx* ctx, size_t region_bytes, uint32_t* placement_out);

/* Mangled symbol of the checksum kernel an attestation of region_bytes at device
 * VA region_va would launch (region_va only decides whether chunk addresses
 * straddle a 4 GiB boundary; 0 = a region that does not), NUL-terminated into
 * buf[buf_len].  Lets a verifier place the running kernel's own machine code in
 * the checksummed region (self-verification; "the beginning of the
 * buffer contains the checksum function itself").  SAGE_EINVAL: invalid
 * region_bytes, NULL buf, buf too small; SAGE_EUNSUPPORTED as for sage_attest. */
int sage_kernel_symbol(sage_ctx* ctx, uint64_t region_va, size_t region_bytes, char* buf, size_t buf_len);

/* The 16-byte UUID of the GPU the context attests (cudaDeviceProp::uuid, the id
 * nvidia-smi prints as GPU-xxxxxxxx-...).  A timing model is a property of one
 * device -- two B200s differ by 0.19% in the median run time of the same kernel,
 * more than the smallest adversary slowdown measured (the
 * paper calibrates per device) -- so a verifier binds its calibration
 * to this id.  SAGE_EINVAL for a NULL argument. */
int sage_device_uuid(sage_ctx* ctx, uint8_t uuid_out[16]);

/* Context and kernel facts (read-only: changes no kernel attribute). */
int sage_query(sage_ctx* ctx, sage_info* out);

/* Number of checksum-kernel launches this context has issued. */
uint64_t sage_launch_count(const sage_ctx* ctx);

/* cudaStream_t the context launches on. */
void* sage_stream(const sage_ctx* ctx);

void sage_checksum_destroy(sage_ctx* ctx);

const char* sage_strerror(int code);
const char* sage_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* SAGE_H */
