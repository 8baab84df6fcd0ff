// variants.cu -- development harness: times lowering variants of the SCS-2
// kernel (the lab form, bench/sage_lab.cuh) at full occupancy on one SMEM/GLOBAL workload and
// checks they all return the same checksum.  Not part of the product path.
//
//   ./variants [rounds] [region_bytes]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "sage_lab.cuh"
namespace sage = sage_lab;

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e = (x);                                                   \
        if (e != cudaSuccess) {                                                \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));            \
            exit(1);                                                           \
        }                                                                      \
    } while (0)

using Fn = void (*)(const sage::KernelArgs);
struct V { const char* name; Fn fn; int P; bool smem; bool straddle; int ilp = 1; int cluster = 0; int stage = 0; int probe = 0; int threads = 1024; };

#define VAR(P, S, ST, XS, U) {"P" #P " smem" #S " straddle" #ST " xs" #XS " unroll" #U, \
                              sage::sage_checksum_kernel<P, S, ST, XS, U>, P, S, ST}
#define VARL(P, LD) {"P" #P " global ld" #LD, sage::sage_checksum_kernel<P, false, true, 0, 1, 0, LD>, P, false, true}
#define VARI(P, U, A, ILP) {"P" #P " smem straddlefalse unroll" #U " addr" #A " ILP" #ILP, \
                           sage::sage_checksum_kernel<P, true, false, 0, U, A, 0, 0, false, 0, ILP>, P, true, false, ILP}
#define VARC(P, U, CL) {"P" #P " cluster-smem unroll" #U " cluster" #CL, \
                        sage::sage_checksum_kernel<P, true, false, 0, U, 3, 0, 0, false, 0, 1>, P, true, false, 1, CL}
#define VARH(P, U, ILP, ST) {"P" #P " hybrid unroll" #U " ILP" #ILP " stage" #ST, \
                           sage::sage_checksum_kernel<P, true, false, 0, U, 7, 0, 0, false, 0, ILP>, P, true, false, ILP, 0, ST}
#define VARG(P, U, ILP) {"P" #P " global unroll" #U " ILP" #ILP, \
                           sage::sage_checksum_kernel<P, false, false, 0, U, 0, 0, 0, false, 0, ILP>, P, false, false, ILP}
#define VARX(P, XS, U, A, ILP) {"P" #P " smem xs" #XS " unroll" #U " addr" #A " ILP" #ILP, \
                           sage::sage_checksum_kernel<P, true, false, XS, U, A, 0, 0, false, 0, ILP>, P, true, false, ILP}
#define VARP(PR) {"P1 smem xs16 unroll32 addr4 PROBE" #PR, \
                  sage::sage_checksum_kernel<1, true, false, 16, 32, 4, 0, 0, false, 0, 1, PR>, 1, true, false, 1, 0, 0, PR}
#define VARQ(U, ILP, PAD, T) {"P1 smem xs16 unroll" #U " addr4 ILP" #ILP " PAD" #PAD " T" #T, \
                  sage::sage_checksum_kernel<1, true, false, 16, U, 4, 0, 0, false, 0, ILP, 0, PAD>, 1, true, false, ILP, 0, 0, 0, T}
#define VARS(U, PR, PAD) {"P1 smem xs16 unroll" #U " addr4 ILP2 PROBE" #PR " PAD" #PAD, \
                  sage::sage_checksum_kernel<1, true, false, 16, U, 4, 0, 0, false, 0, 2, PR, PAD>, 1, true, false, 2}
#define VARGI(P, U, ILP, PAD) {"P" #P " global xs16 unroll" #U " ILP" #ILP " PAD" #PAD, \
                  sage::sage_checksum_kernel<P, false, true, 16, U, 0, 0, 0, false, 0, ILP, 0, PAD>, P, false, true, ILP}
#define VARHP(P, U, ST, PAD) {"P" #P " hybrid unroll" #U " ILP2 stage" #ST " PAD" #PAD, \
                  sage::sage_checksum_kernel<P, true, false, 16, U, 7, 0, 0, false, 0, 2, 0, PAD>, P, true, false, 2, 0, ST}
#define VARH8(U, ST, PAD) {"P1 hybrid8 unroll" #U " ILP2 stage" #ST " PAD" #PAD, \
                  sage::sage_checksum_kernel<1, true, false, 16, U, 8, 0, 0, false, 0, 2, 0, PAD>, 1, true, false, 2, 0, ST}
#define VARA(P, S, ST, XS, U, A) {"P" #P " smem" #S " straddle" #ST " xs" #XS " unroll" #U " addr" #A, \
                              sage::sage_checksum_kernel<P, S, ST, XS, U, A>, P, S, ST}

#define VARY(U, SY) {"P1 smem xs16 unroll" #U " addr4 ILP2 PAD10 SYNC" #SY, \
                  sage::sage_checksum_kernel<1, true, false, 16, U, 4, 0, 0, false, 0, 2, 0, 10, SY>, 1, true, false, 2}

#define VARHS(U, PR, PAD) {"P1 hybrid8 unroll" #U " ILP2 stage196608 PROBE" #PR " PAD" #PAD, \
                  sage::sage_checksum_kernel<1, true, false, 16, U, 8, 0, 0, false, 0, 2, PR, PAD>, 1, true, false, 2, 0, 196608, PR}

// round 2: HBM regions with per-pick L2 eviction priority (LD 5/6, PERSIST_BYTES env)
#define VARGL(P, U, LD) {"P" #P " global xs16 unroll" #U " LD" #LD, \
                  sage::sage_checksum_kernel<P, false, true, 16, U, 0, LD>, P, false, true}
// round 2: hybrid over a 2-CTA cluster (ADDR 9), each CTA stages a different ST bytes
#define VARH9(U, ST, PAD) {"P1 hybrid9 cluster2 unroll" #U " ILP2 stage" #ST " PAD" #PAD, \
                  sage::sage_checksum_kernel<1, true, false, 16, U, 9, 0, 0, false, 0, 2, 0, PAD>, 1, true, false, 2, 2, ST}
// attacker's schedule search: the c2a kernel + EXTRA injected every EVERY rounds
#define VARE(U, PAD, EXTRA, EVERY) {"P1 smem xs16 unroll" #U " addr4 ILP2 PAD" #PAD " EXTRA" #EXTRA " EVERY" #EVERY, \
                  sage::sage_checksum_kernel<1, true, false, 16, U, 4, 0, EXTRA, false, EVERY, 2, 0, PAD>, 1, true, false, 2}
// ... with the xorshift / pick-address lowering searched as well
#define VAREX(XS, U, A, PAD, EXTRA, EVERY) {"P1 smem xs" #XS " unroll" #U " addr" #A " ILP2 PAD" #PAD " EXTRA" #EXTRA \
                  " EVERY" #EVERY, sage::sage_checksum_kernel<1, true, false, XS, U, A, 0, EXTRA, false, EVERY, 2, 0, PAD>, \
                  1, true, false, 2}

// round 2: hybrid (ADDR 8) with the global part's cache operator LD (1 no L1 allocation, 2 .cg)
#define VARH8L(U, ST, PAD, LD) {"P1 hybrid8 unroll" #U " ILP2 stage" #ST " PAD" #PAD " LD" #LD, \
                  sage::sage_checksum_kernel<1, true, false, 16, U, 8, LD, 0, false, 0, 2, 0, PAD>, 1, true, false, 2, 0, ST}
// round 2: pipe-balanced round prototype (BAL extra multiply-adds per round; NOT SCS-2) +
// EXTRA injected (the adversary) every round
#define VARB(U, PAD, BAL, EXTRA) {"P1 smem xs16 unroll" #U " addr4 ILP2 PAD" #PAD " BAL" #BAL " EXTRA" #EXTRA, \
                  sage::sage_checksum_kernel<1, true, false, 16, U, 4, 0, EXTRA, false, 1, 2, 0, PAD, 0, 0, 0, BAL>, \
                  1, true, false, 2, 0, 0, 1}

// round 2 (session 2): the paper buffer at P = 4 / 8 -- hybrid with FMA-pipe addressing (ADDR 10)
#define VARH10(P, U, ILP, ST, PAD) {"P" #P " hybrid10 unroll" #U " ILP" #ILP " stage" #ST " PAD" #PAD, \
                  sage::sage_checksum_kernel<P, true, false, 16, U, 10, 0, 0, false, 0, ILP, 0, PAD>, P, true, false, ILP, 0, ST}

// round 2 (session 2): the P = 1 hybrid with an L1 line prefetch per global pick (ADDR 11, LD 0/1)
#define VARH11(U, ST, PAD, LD) {"P1 hybrid11 unroll" #U " ILP2 stage" #ST " PAD" #PAD " LD" #LD, \
                  sage::sage_checksum_kernel<1, true, false, 16, U, 11, LD, 0, false, 0, 2, 0, PAD>, 1, true, false, 2, 0, ST}

#define VARZ(XS, U, A, PAD) {"P1 smem xs" #XS " unroll" #U " addr" #A " ILP2 PAD" #PAD, \
                  sage::sage_checksum_kernel<1, true, false, XS, U, A, 0, 0, false, 0, 2, 0, PAD>, 1, true, false, 2}

// The list is edited per experiment; the grids behind profiles/r01/variants/*.jsonl were
//   ilp2_grid_u_pad:   VARZ(16, U, 4, PAD) for U in {6,8,10,12,14,16}, PAD in 0..12
//   ilp2_grid2_u_pad:  U in {9,10,11,13,15,18,20}, PAD in 0..12
//   ilp2_grid3_u_pad:  U in {17,18,19,21,22,24,26,28,32}, PAD in 4..10
//   ilp2_order_sweep:  VARS(U, 16, PAD) for U in {8,10,12,14,16,17,18,20}, PAD in {0,4..10}
//   hybrid_u_pad:      VARH8(U, 196608, PAD) for U in {1,2,3,4,6}, PAD in {0,2,4..10} (region 524288)
//   sync_sweep:        VARY(16, SYNC) for SYNC in {0,1,4,16,64,256}
//   ilp4_grid_u_pad:   VARQ(U, 4, PAD, 512) for U in {2,3,4,6,8}, PAD in {0,8,14..24 step 2}
//   ilp2_t512_sweep:   VARQ(U, 2, PAD, 512) for U in {16,17,18}, PAD in {0,6,7,8,10}
//   ilp2_xs_sweep:     VARZ(XS, U, 4, PAD) for XS in {17,18,20}, U in {16,17,18}, PAD in {0,5,6,7,8,10}
//   hybrid_stage_sweep: VARH8(2, STAGE, 8) for STAGE in 160..212 KiB (region 524288)
//   hybrid_stagger:    VARHS(U, PROBE, PAD) for PROBE in {4, 12} (region 524288)
// Default: the current product kernels and their nearest alternatives.
static V variants[] = {
#ifdef VARIANTS_INC
#include VARIANTS_INC          // a generated list (scripts/schedule_search.py)
#else
    VARZ(16, 18, 4, 7), VARZ(16, 16, 4, 10), VARZ(16, 18, 4, 0), VARZ(16, 18, 4, 8), VARZ(16, 17, 4, 7),
    VARH8(2, 196608, 8), VARZ(16, 18, 4, 7),
#endif
};

int main(int argc, char** argv) {
    const uint32_t rounds = argc > 1 ? atoi(argv[1]) : 100000;
    const size_t bytes = argc > 2 ? strtoull(argv[2], nullptr, 10) : 8192;
    const int gran = argc > 3 ? atoi(argv[3]) : -1;
    size_t cur = 0;
    CK(cudaDeviceGetLimit(&cur, cudaLimitMaxL2FetchGranularity));
    if (gran >= 0) CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran));
    size_t now = 0;
    CK(cudaDeviceGetLimit(&now, cudaLimitMaxL2FetchGranularity));
    fprintf(stderr, "L2 fetch granularity default %zu now %zu\n", cur, now);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int blocks = 2 * sms, threads = 1024;
    std::vector<uint8_t> h(bytes);
    srand(7);
    for (auto& b : h) b = rand() & 0xFF;
    uint8_t* d = nullptr;
    CK(cudaMalloc(&d, bytes));
    CK(cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice));
    uint64_t* raw = nullptr;
    CK(cudaMalloc(&raw, 32));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const bool straddles = (reinterpret_cast<uint64_t>(d) >> 32) != ((reinterpret_cast<uint64_t>(d) + bytes - 1) >> 32);
    unsigned long long ref[9] = {0};
    const char* only = argc > 4 ? argv[4] : nullptr;
    // round 2 (env): PERSIST_BYTES for LD 5/6 kernels; WINDOW_BYTES / HIT_RATIO: an L2
    // access-policy window (persisting hits, streaming misses) over the region's first
    // WINDOW_BYTES, with the persisting carve-out set to its maximum
    const uint64_t persist_bytes = getenv("PERSIST_BYTES") ? strtoull(getenv("PERSIST_BYTES"), nullptr, 10) : 0;
    cudaStream_t st = nullptr;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    if (getenv("WINDOW_BYTES")) {
        int maxp = 0, maxw = 0;
        CK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0));
        CK(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, 0));
        CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, maxp));
        size_t setp = 0;
        CK(cudaDeviceGetLimit(&setp, cudaLimitPersistingL2CacheSize));
        cudaStreamAttrValue av = {};
        size_t wb = strtoull(getenv("WINDOW_BYTES"), nullptr, 10);
        if (wb > (size_t)maxw) wb = maxw;
        av.accessPolicyWindow.base_ptr = d;
        av.accessPolicyWindow.num_bytes = wb;
        av.accessPolicyWindow.hitRatio = getenv("HIT_RATIO") ? atof(getenv("HIT_RATIO")) : 1.0f;
        av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
        fprintf(stderr, "{\"max_persisting_l2\": %d, \"persisting_limit_set\": %zu, \"max_window\": %d, "
                "\"window_bytes\": %zu, \"hit_ratio\": %.3f}\n", maxp, setp, maxw, wb, av.accessPolicyWindow.hitRatio);
    } else if (persist_bytes) {
        int maxp = 0;
        CK(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0));
        if (!getenv("NO_PERSIST_LIMIT")) CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, maxp));
        fprintf(stderr, "{\"max_persisting_l2\": %d, \"persist_bytes\": %llu}\n", maxp,
                (unsigned long long)persist_bytes);
    }
    for (auto& v : variants) {
        if (only && strstr(v.name, only) == nullptr) continue;
        if (!v.straddle && straddles) continue;
        size_t dyn = v.smem ? bytes : 0;
        if (v.stage) {
            if ((size_t)v.stage >= bytes) continue;
            dyn = v.stage;
        } else if (v.cluster) {
            dyn = bytes / v.cluster;
            if (dyn > 65536 || dyn < 16) continue;
        } else if (v.smem && bytes > 65536) continue;
        if (v.smem) CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(v.fn),
                                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn));
        if (getenv("CARVEOUT"))
            CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(v.fn), cudaFuncAttributePreferredSharedMemoryCarveout,
                                    atoi(getenv("CARVEOUT"))));
        sage::KernelArgs a{};
        a.region = reinterpret_cast<const uint32_t*>(d);
        a.nonce = 0x1234;
        a.nc_mask = uint32_t(bytes / (4 * v.P) - 1);
        a.rounds = rounds;
        a.region_bytes = uint32_t(dyn);
        a.slice_shift = 0;
        while ((size_t(1) << a.slice_shift) < dyn) ++a.slice_shift;
        a.raw = raw;
        a.persist_bytes = persist_bytes;
        sage::fill_tables(a, v.P);
        const int grid = blocks * threads / (v.ilp * v.threads);
        if (v.cluster) {
            cudaLaunchConfig_t occ = {};
            occ.gridDim = dim3(grid);
            occ.blockDim = dim3(v.threads);
            occ.dynamicSmemBytes = dyn;
            cudaLaunchAttribute oat[1];
            oat[0].id = cudaLaunchAttributeClusterDimension;
            oat[0].val.clusterDim.x = v.cluster;
            oat[0].val.clusterDim.y = 1;
            oat[0].val.clusterDim.z = 1;
            occ.attrs = oat;
            occ.numAttrs = 1;
            int nclusters = 0;
            if (cudaOccupancyMaxActiveClusters(&nclusters, v.fn, &occ) == cudaSuccess)
                fprintf(stderr, "{\"variant\": \"%s\", \"max_active_clusters\": %d, \"clusters_needed\": %d}\n",
                        v.name, nclusters, grid / v.cluster);
            else
                cudaGetLastError();
        }
        float best = 1e30f;
        unsigned long long h_raw[4];
        for (int rep = 0; rep < 3; ++rep) {
            CK(cudaMemsetAsync(raw, 0, 32, st));
            CK(cudaEventRecord(e0, st));
            if (v.cluster) {
                cudaLaunchConfig_t cfg = {};
                cfg.stream = st;
                cfg.gridDim = dim3(grid);
                cfg.blockDim = dim3(threads);
                cfg.dynamicSmemBytes = dyn;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = v.cluster;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                CK(cudaLaunchKernelEx(&cfg, v.fn, a));
            } else {
                v.fn<<<grid, v.threads, dyn, st>>>(a);
            }
            CK(cudaEventRecord(e1, st));
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < best) best = ms;
            CK(cudaMemcpy(h_raw, raw, 32, cudaMemcpyDeviceToHost));
        }
        if (ref[v.P] == 0 && v.probe == 0) ref[v.P] = h_raw[0];
        const double tr = double(blocks) * threads * rounds / (best * 1e-3);
        printf("{\"variant\": \"%s\", \"ms\": %.3f, \"thread_rounds_per_s\": %.4e, \"cycles\": %llu, "
               "\"cycles_per_round\": %.1f, \"checksum\": \"0x%016llx\", \"same\": %s}\n",
               v.name, best, tr, h_raw[1], double(h_raw[1]) / rounds, h_raw[0], h_raw[0] == ref[v.P] ? "true" : "false");
        fflush(stdout);
    }
    return 0;
}
