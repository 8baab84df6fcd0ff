// stall_trace.cu -- diagnostics for the attestation-time slow mode:
// runs the product's c2a kernel with a per-CTA progress trace (PROBE bit 5: thread 0
// of every CTA stamps %globaltimer every EVERY trips of 18 rounds) and reports, per
// run, the intervals that are longer than the CTA's median interval by more than
// 300 us, grouped into events by start time.  A chip-wide stall shows up as one
// event on (nearly) every CTA at the same time with the same excess.
//   ./stall_trace [rounds=1000000] [runs=20] [every=32] > stalls.jsonl
#include <cuda_runtime.h>

#include <algorithm>
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

int main(int argc, char** argv) {
    const uint32_t rounds = argc > 1 ? atoi(argv[1]) : 1000000;
    const int runs = argc > 2 ? atoi(argv[2]) : 20;
    const uint32_t every = argc > 3 ? atoi(argv[3]) : 32;
    auto fn = sage::sage_checksum_kernel<1, true, false, 16, 18, 4, 0, 0, false, 0, 2, 32, 7>;
    const size_t bytes = 8192;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int ctas = sms;                                  // ILP 2: one CTA of 1024 threads per SM
    std::vector<uint8_t> h(bytes);
    srand(5);
    for (auto& b : h) b = rand() & 0xFF;
    uint8_t* d = nullptr;
    CK(cudaMalloc(&d, bytes));
    CK(cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice));
    uint64_t* raw = nullptr;
    CK(cudaMalloc(&raw, 32));
    const uint32_t trips = rounds / 18;
    const uint32_t slots = trips / every + 1;
    uint64_t* prog = nullptr;
    CK(cudaMalloc(&prog, sizeof(uint64_t) * slots * ctas));
    std::vector<uint64_t> hp(size_t(slots) * ctas);
    CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    sage::KernelArgs a{};
    a.region = reinterpret_cast<const uint32_t*>(d);
    a.nonce = 0x57A11;
    a.nc_mask = uint32_t(bytes / 4 - 1);
    a.rounds = rounds;
    a.region_bytes = uint32_t(bytes);
    a.raw = raw;
    a.progress = prog;
    a.progress_every = every;
    a.progress_slots = slots;
    sage::fill_tables(a, 1);
    for (int run = -2; run < runs; ++run) {
        CK(cudaMemset(raw, 0, 32));
        CK(cudaMemset(prog, 0, sizeof(uint64_t) * slots * ctas));
        fn<<<ctas, 1024, bytes>>>(a);
        CK(cudaDeviceSynchronize());
        if (run < 0) continue;
        uint64_t hr[4];
        CK(cudaMemcpy(hr, raw, 32, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(hp.data(), prog, hp.size() * 8, cudaMemcpyDeviceToHost));
        const uint64_t t0 = ~hr[2];
        // per-CTA long intervals
        struct Gap { int cta; double start_ms, excess_us; };
        std::vector<Gap> gaps;
        double med_all = 0;
        for (int c = 0; c < ctas; ++c) {
            std::vector<double> iv;
            for (uint32_t k = 1; k < slots; ++k) {
                const uint64_t x0 = hp[size_t(c) * slots + k - 1], x1 = hp[size_t(c) * slots + k];
                if (x0 && x1) iv.push_back(double(x1 - x0));
            }
            if (iv.empty()) continue;
            std::vector<double> srt = iv;
            std::sort(srt.begin(), srt.end());
            const double med = srt[srt.size() / 2];
            med_all += med / ctas;
            for (uint32_t k = 1; k < slots; ++k) {
                const uint64_t x0 = hp[size_t(c) * slots + k - 1], x1 = hp[size_t(c) * slots + k];
                if (!x0 || !x1) continue;
                const double ex = double(x1 - x0) - med;
                if (ex > 300e3) gaps.push_back({c, (x0 - t0) / 1e6, ex / 1e3});
            }
        }
        std::sort(gaps.begin(), gaps.end(), [](const Gap& p, const Gap& q) { return p.start_ms < q.start_ms; });
        // group into events: gaps whose start times lie within one interval of each other
        printf("{\"run\": %d, \"rounds\": %u, \"device_ms\": %.3f, \"cycles\": %llu, \"interval_us\": %.1f, \"events\": [",
               run, rounds, (hr[3] - t0) / 1e6, (unsigned long long)hr[1], med_all / 1e3);
        size_t i = 0;
        bool first = true;
        while (i < gaps.size()) {
            size_t j = i;
            double ex_sum = 0, ex_min = 1e30, ex_max = 0;
            while (j < gaps.size() && gaps[j].start_ms - gaps[i].start_ms < 2.0 * med_all / 1e6 + 0.5) {
                ex_sum += gaps[j].excess_us;
                ex_min = std::min(ex_min, gaps[j].excess_us);
                ex_max = std::max(ex_max, gaps[j].excess_us);
                ++j;
            }
            printf("%s{\"t_ms\": %.3f, \"ctas\": %zu, \"excess_us_mean\": %.1f, \"min\": %.1f, \"max\": %.1f}",
                   first ? "" : ", ", gaps[i].start_ms, j - i, ex_sum / (j - i), ex_min, ex_max);
            first = false;
            i = j;
        }
        printf("]}\n");
        fflush(stdout);
    }
    return 0;
}
