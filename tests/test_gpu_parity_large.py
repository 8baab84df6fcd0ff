"""GPU parity at the largest configurations: the 2 GiB HBM regions
(bench configs c3big / c3bigp8) at full occupancy, and a config-4 attestation at
R = 10^7 -- sampled warps recomputed by the oracle plus sum consistency -- and the
inclusion experiment's read counts compared chunk by chunk with the oracle's
(integer index work: bit-exact)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle                                                     # noqa: E402
from paper_2209_03125_b200 import sage                            # noqa: E402
from paper_2209_03125_b200.inputs import launched_kernel_prefix, make_region, nonces  # noqa: E402

pytestmark = pytest.mark.gpu
M64 = (1 << 64) - 1


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2209_03125_b200 import build
    build.build()
    return torch.device("cuda:0")


@pytest.mark.parametrize("P", [1, 8])
def test_2gib_hbm_region_full_occupancy(dev, P):
    """c3big (P = 1) and c3bigp8 (P = 8) as bench.py times them: 2 GiB region in HBM
    (GLOBAL), full occupancy, R = 10^4 (BASELINE configs[2]); the per-warp partials
    sum to the checksum and 4 sampled warps (first, last, two inside) equal the
    oracle's on the same bytes and device VA."""
    nbytes = 2 << 30
    g = torch.Generator(device=dev)
    g.manual_seed(0x5EED0001 + P)
    d = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=dev, generator=g)
    R = 10_000
    nonce = nonces(3)[P % 3]
    with sage.Context(pick_words=P) as ctx:
        info = ctx.query()
        n = info.blocks * info.threads
        pw = torch.zeros(n // 32, dtype=torch.int64, device=dev)
        res = ctx.attest_debug(nonce, d, R, pw)
    assert res.placement == sage.SAGE_GLOBAL
    parts = [int(v) & M64 for v in pw.cpu().tolist()]
    assert sum(parts) & M64 == res.checksum
    region = d.cpu().numpy()
    for w in (0, 1234, n // 64 + 7, n // 32 - 1):
        assert parts[w] == oracle.warp_sum(nonce, region, d.data_ptr(), R, w, P), w
    del d


def test_config4_longest_attestation_sampled(dev):
    """Config 4's longest round count, R = 10^7 (~5.4 s on the GPU), at the bench
    geometry (full occupancy, 8 KiB SMEM region of the kernel's own code): sum of
    partials == checksum, and one warp recomputed by the oracle (~5 s of CPU)."""
    region = make_region(8192, prefix=launched_kernel_prefix(8192))
    d = torch.from_numpy(region).to(dev)
    R = 10_000_000
    nonce = nonces(5)[4]
    with sage.Context() as ctx:
        info = ctx.query()
        n = info.blocks * info.threads
        pw = torch.zeros(n // 32, dtype=torch.int64, device=dev)
        res = ctx.attest_debug(nonce, d, R, pw)
    parts = [int(v) & M64 for v in pw.cpu().tolist()]
    assert sum(parts) & M64 == res.checksum
    w = 4097
    assert parts[w] == oracle.warp_sum(nonce, region, d.data_ptr(), R, w, 1)


@pytest.mark.parametrize("blocks,threads,words,rounds,P", [
    (1, 32, 131072, 3125, 1),          # P:748's experiment: N = 100,000 picks
    (1, 32, 524288, 3125, 1),
    (4, 256, 16384, 100, 4),
    (0, 0, 131072, 16, 1),             # full occupancy: every word read
])
def test_coverage_counts_bit_exact(dev, blocks, threads, words, rounds, P):
    """sage_attest_coverage's per-chunk read counts equal the oracle's count of the
    same attestation's picks for every chunk, and its
    checksum equals the oracle's."""
    region = make_region(4 * words, fill_seed=words + P)
    d = torch.from_numpy(region).to(dev)
    counts = torch.zeros(words // P, dtype=torch.int32, device=dev)
    with sage.Context(blocks=blocks, threads=threads, pick_words=P) as ctx:
        info = ctx.query()
        res = ctx.attest_coverage(0xC0FFEE + P, d, rounds, counts)
    want_sum, want = oracle.attest_counts(0xC0FFEE + P, region, d.data_ptr(), rounds, info.blocks, info.threads, P)
    assert res.checksum == want_sum
    got = counts.cpu().numpy().astype(np.uint32)
    assert np.array_equal(got, want), int((got != want).sum())
    assert int(got.sum()) == info.blocks * info.threads * rounds
