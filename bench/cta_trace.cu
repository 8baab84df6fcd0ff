// cta_trace.cu -- diagnostics for the attestation-time tail:
// runs the product's c2a kernel many times and dumps, per run, every CTA's
// SM id, start/end %globaltimer and clock64 span.
//   ./cta_trace [rounds=100000] [runs=200] > trace.jsonl
#include <cuda_runtime.h>

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
    const uint32_t rounds = argc > 1 ? atoi(argv[1]) : 100000;
    const int runs = argc > 2 ? atoi(argv[2]) : 200;
    const size_t bytes = 8192;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int blocks = 2 * sms, threads = 1024;
    std::vector<uint8_t> h(bytes);
    for (size_t i = 0; i < bytes; ++i) h[i] = uint8_t(i * 131 + 7);
    uint8_t* d;
    CK(cudaMalloc(&d, bytes));
    CK(cudaMemcpy(d, h.data(), bytes, cudaMemcpyHostToDevice));
    uint64_t *raw, *tr;
    CK(cudaMalloc(&raw, 32));
    CK(cudaMalloc(&tr, 32ull * blocks));
    auto fn = sage::sage_checksum_kernel<1, true, false, 0, 32, 1, 0, 0>;
    CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    sage::KernelArgs a{};
    a.region = reinterpret_cast<const uint32_t*>(d);
    a.nc_mask = uint32_t(bytes / 4 - 1);
    a.rounds = rounds;
    a.region_bytes = uint32_t(bytes);
    a.raw = raw;
    a.cta_trace = tr;
    sage::fill_tables(a, 1);
    std::vector<uint64_t> ht(4ull * blocks);
    uint64_t hraw[4];
    for (int r = 0; r < runs; ++r) {
        a.nonce = 1000 + r;
        CK(cudaMemset(raw, 0, 32));
        fn<<<blocks, threads, bytes>>>(a);
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(ht.data(), tr, 32ull * blocks, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(hraw, raw, 32, cudaMemcpyDeviceToHost));
        printf("{\"run\": %d, \"cycles\": %llu, \"cta\": [", r, (unsigned long long)hraw[1]);
        for (int b = 0; b < blocks; ++b)
            printf("%s[%llu,%llu,%llu,%llu]", b ? "," : "", (unsigned long long)ht[4 * b], (unsigned long long)ht[4 * b + 1],
                   (unsigned long long)ht[4 * b + 2], (unsigned long long)ht[4 * b + 3]);
        printf("]}\n");
    }
    return 0;
}
