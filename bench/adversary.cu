// adversary.cu -- Table 1 Exp 1 vs Exp 2 on B200.
//
// The paper measures the honest checksum 100 times (T_avg, sigma), sets the
// detection threshold at T_avg + 2.5 sigma, then inserts ONE extra
// instruction into the checksum loop and shows that even its fastest run
// T_min exceeds the threshold (Table 1).  Here the
// honest kernel is the product's c2a kernel (full occupancy, 8 KiB SMEM
// region, P=1) and each adversary is the same kernel with EXTRA
// result-neutral dependent ALU instructions injected once every UNROLL
// rounds (so it still returns the correct checksum).  Timing is the
// verifier's: host CLOCK_MONOTONIC from before the launch to the result on
// the host (as in sage_attest); the kernels are interleaved run by run.
// One JSON line per kernel, then a summary per honest/adversary pair.
//
//   ./adversary [rounds=100000] [runs=100]
#include <cuda_runtime.h>
#include <time.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
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
struct K { const char* name; Fn fn; int extra; int every; int ilp = 1; };

// <P, SMEM, STRADDLE, XS, UNROLL, ADDR, LD, EXTRA, COUNT, EVERY, ILP, PROBE, PAD, SYNC, FEXTRA>;
// the honest kernel is the product's c2a kernel (XS 16, UNROLL 18, ADDR 4, ILP 2, PAD 7)
static K kernels[] = {
    {"honest", sage::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, 0, false, 0, 2, 0, 7>, 0, 0, 2},
    {"+1 instr / round", sage::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, 1, false, 1, 2, 0, 7>, 1, 1, 2},
    {"+1 instr / 9 rounds", sage::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, 1, false, 9, 2, 0, 7>, 1, 9, 2},
    {"+1 instr / 18 rounds", sage::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, 1, false, 18, 2, 0, 7>, 1, 18, 2},
    {"+1 IMAD / round", sage::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, -1, false, 1, 2, 0, 7>, -1, 1, 2},
    {"+2 IMAD / round", sage::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, -2, false, 1, 2, 0, 7>, -2, 1, 2},
    // other implementations of the same function an adversary could switch to:
    // the ILP 1 kernel (2 CTAs x 1024 threads per SM, 32 registers; the previous
    // product) and the ILP 2 kernel without the register reservation (56 registers)
    {"ILP1 (2 CTAs/SM)", sage::sage_checksum_kernel<1, true, false, 16, 32, 4, 0, 0>, 0, 0, 1},
    {"ILP1 +1 IMAD / round", sage::sage_checksum_kernel<1, true, false, 16, 32, 4, 0, -1, false, 1>, -1, 1, 1},
    {"ILP2 U16 PAD10 (previous product)", sage::sage_checksum_kernel<1, true, false, 16, 16, 4, 0, 0, false, 0, 2, 0, 10>, 0, 0, 2},
    {"ILP2 U18 unpadded", sage::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, 0, false, 0, 2>, 0, 0, 2},
    {"ILP2 U18 unpadded +1 IMAD / round", sage::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, -1, false, 1, 2>, -1, 1, 2},
    {"ILP2 unpadded", sage::sage_checksum_kernel<1, true, false, 16, 16, 4, 0, 0, false, 0, 2>, 0, 0, 2},
    {"ILP2 unpadded +1 IMAD / round", sage::sage_checksum_kernel<1, true, false, 16, 16, 4, 0, -1, false, 1, 2>, -1, 1, 2},
    {"ILP2 unpadded +1 instr / 16", sage::sage_checksum_kernel<1, true, false, 16, 16, 4, 0, 1, false, 16, 2>, 1, 16, 2},
    // the adversary's own work in the issue slots the checksum leaves idle: a chain
    // independent of the checksum state, FP32 FFMA (FEXTRA > 0) or integer IMAD (< 0)
    {"+1 indep FFMA / round", sage::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, 0, false, 0, 2, 0, 7, 0, 1>, 0, 1, 2},
    {"+2 indep FFMA / round", sage::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, 0, false, 0, 2, 0, 7, 0, 2>, 0, 1, 2},
    {"+4 indep FFMA / round", sage::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, 0, false, 0, 2, 0, 7, 0, 4>, 0, 1, 2},
    {"+8 indep FFMA / round", sage::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, 0, false, 0, 2, 0, 7, 0, 8>, 0, 1, 2},
    {"+1 indep IMAD / round", sage::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, 0, false, 0, 2, 0, 7, 0, -1>, 0, 1, 2},
};

static uint64_t now_ns() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return uint64_t(ts.tv_sec) * 1000000000ull + uint64_t(ts.tv_nsec);
}

int main(int argc, char** argv) {
    const uint32_t rounds = argc > 1 ? atoi(argv[1]) : 100000;
    const int runs = argc > 2 ? atoi(argv[2]) : 100;
    const size_t bytes = 8192;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int blocks = 2 * sms, threads = 1024;
    std::vector<uint8_t> h(bytes);
    srand(11);
    for (auto& b : h) b = rand() & 0xFF;
    uint8_t* d = nullptr;
    CK(cudaMalloc(&d, bytes));
    CK(cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice));
    uint64_t *raw = nullptr, *hraw = nullptr;
    CK(cudaMalloc(&raw, 32));
    CK(cudaMallocHost(&hraw, 32));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    struct Stat { double avg, sd, mn, mx, med, mad; uint64_t cs; std::vector<double> t; };
    std::vector<Stat> st;
    // all kernels interleaved run by run, so drift (clocks, temperature) hits them alike
    const int nk = sizeof(kernels) / sizeof(kernels[0]);
    std::vector<sage::KernelArgs> args(nk);
    std::vector<std::vector<double>> times(nk);
    std::vector<uint64_t> sums(nk, 0);
    for (int j = 0; j < nk; ++j) {
        CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(kernels[j].fn),
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        sage::KernelArgs& a = args[j];
        a = sage::KernelArgs{};
        a.region = reinterpret_cast<const uint32_t*>(d);
        a.nonce = 0xA77E57;
        a.nc_mask = uint32_t(bytes / 4 - 1);
        a.rounds = rounds;
        a.region_bytes = uint32_t(bytes);
        a.raw = raw;
        sage::fill_tables(a, 1);
    }
    for (int i = -3; i < runs; ++i) {           // 3 warm-up passes
        for (int j = 0; j < nk; ++j) {
            const uint64_t t0 = now_ns();
            CK(cudaMemsetAsync(raw, 0, 32, s));
            kernels[j].fn<<<blocks / kernels[j].ilp, threads, bytes, s>>>(args[j]);
            CK(cudaMemcpyAsync(hraw, raw, 32, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            const uint64_t t1 = now_ns();
            if (i >= 0) times[j].push_back((t1 - t0) * 1e-9);
            sums[j] = hraw[0];
        }
    }
    for (int j = 0; j < nk; ++j) {
        const auto& k = kernels[j];
        const std::vector<double>& t = times[j];
        const uint64_t cs = sums[j];
        double m = 0, v = 0;
        for (double x : t) m += x;
        m /= t.size();
        for (double x : t) v += (x - m) * (x - m);
        v /= t.size();
        std::vector<double> srt = t;
        std::sort(srt.begin(), srt.end());
        const double med = srt[srt.size() / 2];
        std::vector<double> dev;
        for (double x : t) dev.push_back(std::fabs(x - med));
        std::sort(dev.begin(), dev.end());
        Stat q{m, std::sqrt(v), srt.front(), srt.back(), med, dev[dev.size() / 2], cs, t};
        st.push_back(q);
        printf("{\"kernel\": \"%s\", \"extra_instr\": %d, \"every_rounds\": %d, \"runs\": %d, \"t_avg_s\": %.6f, "
               "\"sigma_s\": %.6f, \"t_min_s\": %.6f, \"t_med_s\": %.6f, \"t_max_s\": %.6f, \"threshold_s\": %.6f, "
               "\"checksum\": \"0x%016llx\"}\n",
               k.name, k.extra, k.every, runs, q.avg, q.sd, q.mn, q.med, q.mx, q.avg + 2.5 * q.sd, (unsigned long long)cs);
        fflush(stdout);
    }
    // verdicts: adversary vs the honest kernel with the same unroll
    for (int jj = 1; jj < nk; ++jj) {
        const int p[2] = {0, jj};
        const Stat& hs = st[p[0]];
        const Stat& as = st[p[1]];
        // calibrate on the first half of the honest runs, evaluate on the second half
        const size_t half = hs.t.size() / 2;
        std::vector<double> cal(hs.t.begin(), hs.t.begin() + half), held(hs.t.begin() + half, hs.t.end());
        double cm = 0, cv = 0;
        for (double x : cal) cm += x;
        cm /= cal.size();
        for (double x : cal) cv += (x - cm) * (x - cm);
        cv = std::sqrt(cv / cal.size());
        const double thr = cm + 2.5 * cv;                              // the paper's rule
        // empirical-quantile rule: the calibration runs' 99th percentile
        std::vector<double> csrt = cal;
        std::sort(csrt.begin(), csrt.end());
        const double rthr = csrt[size_t(0.99 * (csrt.size() - 1))];
        const double qthr = csrt[size_t(0.95 * (csrt.size() - 1))];   // restart policy threshold
        // robust relative rule (verifier.calibrate_robust): median * (1 + max(5e-3, 6 * 1.4826 * MAD / median))
        const double cmed = csrt[csrt.size() / 2];
        std::vector<double> cdev;
        for (double x : cal) cdev.push_back(std::fabs(x - cmed));
        std::sort(cdev.begin(), cdev.end());
        const double bthr = cmed * (1.0 + std::max(5e-3, 6.0 * 1.4826 * cdev[cdev.size() / 2] / cmed));
        auto frac_above = [](const std::vector<double>& xs, double th) {
            size_t c = 0;
            for (double x : xs) c += x > th;
            return double(c) / xs.size();
        };
        printf("{\"summary\": \"%s vs %s\", \"rounds\": %u, \"honest_t_avg_s\": %.6f, \"honest_sigma_s\": %.6f, "
               "\"threshold_s\": %.6f, \"adversary_t_min_s\": %.6f, \"adversary_t_med_s\": %.6f, \"slowdown\": %.5f, "
               "\"detected_tmin_gt_threshold\": %s, \"honest_rejected_frac\": %.3f, \"adversary_rejected_frac\": %.3f, "
               "\"p99_threshold_s\": %.6f, \"p99_honest_rejected_frac\": %.3f, \"p99_adversary_rejected_frac\": %.3f, "
               "\"p95_threshold_s\": %.6f, \"p95_honest_reject_per_try\": %.3f, \"p95_adversary_accept_per_try\": %.3f, "
               "\"robust_threshold_s\": %.6f, \"robust_honest_reject_per_try\": %.3f, "
               "\"robust_adversary_rejected_frac\": %.3f, \"same_checksum\": %s}\n",
               kernels[p[1]].name, kernels[p[0]].name, rounds, cm, cv, thr, as.mn, as.med, as.med / hs.med - 1.0,
               as.mn > thr ? "true" : "false", frac_above(held, thr), frac_above(as.t, thr), rthr,
               frac_above(held, rthr), frac_above(as.t, rthr), qthr, frac_above(held, qthr), 1.0 - frac_above(as.t, qthr),
               bthr, frac_above(held, bthr), frac_above(as.t, bthr), hs.cs == as.cs ? "true" : "false");
    }
    return 0;
}
