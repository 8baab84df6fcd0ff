/*
 * attest_cli.c -- the C ABI used from plain C (no Python, no torch):
 * allocate a region, fill it, attest it with a nonce, print the result.
 *
 *   gcc -O2 -I include examples/attest_cli.c -o attest_cli \
 *       -L paper_2209_03125_b200 -lsage -Wl,-rpath,$PWD/paper_2209_03125_b200
 *   ./attest_cli [rounds] [region_bytes] [nonce]
 *
 * Output: one JSON line with the checksum, cycles, host elapsed and device ns.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "sage.h"

int main(int argc, char** argv) {
    const uint64_t rounds = argc > 1 ? strtoull(argv[1], NULL, 10) : 100000;
    const size_t bytes = argc > 2 ? strtoull(argv[2], NULL, 10) : 8192;
    const uint64_t nonce = argc > 3 ? strtoull(argv[3], NULL, 0) : 0x0123456789ABCDEFull;

    sage_ctx* ctx = NULL;
    int rc = sage_checksum_init(NULL, &ctx);               /* full occupancy on device 0 */
    if (rc) { fprintf(stderr, "init: %s (%s)\n", sage_strerror(rc), sage_last_error()); return 1; }

    /* host region: a deterministic byte pattern; attested through the host path,
     * which stages it in a context-owned device buffer whose VA it reports */
    unsigned char* host = (unsigned char*)malloc(bytes);
    if (!host) return 1;
    for (size_t i = 0; i < bytes; ++i) host[i] = (unsigned char)(i * 2654435761u >> 13);

    sage_result res;
    rc = sage_attest_host(ctx, nonce, host, bytes, rounds, &res);
    if (rc) { fprintf(stderr, "attest: %s (%s)\n", sage_strerror(rc), sage_last_error()); return 1; }
    printf("{\"checksum\": \"0x%016llx\", \"cycles\": %llu, \"elapsed_ns\": %llu, \"device_ns\": %llu, "
           "\"region_va\": \"0x%llx\", \"placement\": %u, \"blocks\": %u, \"threads\": %u}\n",
           (unsigned long long)res.checksum, (unsigned long long)res.cycles, (unsigned long long)res.elapsed_ns,
           (unsigned long long)res.device_ns, (unsigned long long)res.region_va, res.placement, res.blocks,
           res.threads);
    free(host);
    sage_checksum_destroy(ctx);
    return 0;
}
