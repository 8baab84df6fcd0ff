"""GPU parity: the sm_100a kernel behind libsage.so against the CPU oracle,
bit-exact (integer work).  Every call goes through the C ABI (ctypes binding).
The oracle receives the region's real device VA (the data pointer is folded
in every round)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle                                                     # noqa: E402
from paper_2209_03125_b200 import sage                            # noqa: E402
from paper_2209_03125_b200.inputs import (C1_NONCE, launched_kernel_prefix, make_region,  # noqa: E402
                                           nonces)

pytestmark = pytest.mark.gpu

M64 = (1 << 64) - 1


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2209_03125_b200 import build
    build.build()
    return torch.device("cuda:0")


def to_dev(region_np, dev, align_offset=0):
    """Copy a host region to a fresh device buffer at a given byte offset (>= 0,
    multiple of 16) from a 256-B aligned allocation; returns (tensor_view, keepalive)."""
    n = region_np.nbytes
    buf = torch.empty(n + align_offset + 256, dtype=torch.uint8, device=dev)
    start = (-buf.data_ptr()) % 256 + align_offset
    view = buf[start:start + n]
    view.copy_(torch.from_numpy(region_np))
    assert view.data_ptr() % 16 == 0
    return view, buf


def test_config1_bit_exact(dev):
    """BASELINE configs[0]: 1 x 32 threads, 4 KiB region, 10^4 rounds, fixed nonce."""
    region = make_region(4096, prefix=launched_kernel_prefix(4096, blocks=1, threads=32))
    d, _keep = to_dev(region, dev)
    with sage.Context(blocks=1, threads=32) as ctx:
        res = ctx.attest(C1_NONCE, d, 10_000)
        assert res.placement == sage.SAGE_SMEM
        want = oracle.attest(C1_NONCE, region, d.data_ptr(), 10_000, 1, 32, 1)
        assert res.checksum == want
        assert res.cycles > 0 and res.elapsed_ns > 0 and res.device_ns > 0


@pytest.mark.parametrize("seed", range(6))
def test_random_small_geometries(dev, seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(8):
        P = int(rng.choice([1, 4, 8]))
        nc = 1 << int(rng.integers(0, 12))
        nbytes = 4 * P * nc
        if nbytes < 16:
            P, nc, nbytes = 1, 4, 16
        placement = int(rng.choice([sage.SAGE_AUTO, sage.SAGE_SMEM, sage.SAGE_GLOBAL]))
        blocks = int(rng.integers(1, 5))
        threads = 32 * int(rng.integers(1, 9))
        rounds = int(rng.integers(0, 400))
        nonce = int(rng.integers(0, 2**64, dtype=np.uint64))
        region = make_region(nbytes, fill_seed=int(rng.integers(0, 2**31)))
        d, _keep = to_dev(region, dev, align_offset=32 * int(rng.integers(0, 8)))
        pw = torch.zeros(blocks * threads // 32, dtype=torch.int64, device=dev)
        with sage.Context(blocks=blocks, threads=threads, pick_words=P, placement=placement) as ctx:
            res = ctx.attest_debug(nonce, d, rounds, pw)
        want = oracle.attest(nonce, region, d.data_ptr(), rounds, blocks, threads, P)
        assert res.checksum == want, dict(P=P, nc=nc, placement=placement, blocks=blocks, threads=threads,
                                          rounds=rounds)
        parts = [int(v) & M64 for v in pw.cpu().tolist()]
        w = int(rng.integers(0, len(parts)))
        assert parts[w] == oracle.warp_sum(nonce, region, d.data_ptr(), rounds, w, P)


@pytest.mark.parametrize("seed", range(3))
def test_random_ilp2_geometries(dev, seed):
    """Random cases at the ILP-2 geometry (1024-thread blocks, even block count: the
    c2a SMEM kernel and the P = 1 / 4 SAGE_HYBRID kernels): random P in {1, 4},
    region size (16 B ... 1 MiB; HYBRID stages min(region, 192 KiB)), placement
    (AUTO, SMEM where it fits, HYBRID, GLOBAL), rounds (0 ... 300, covering the
    unrolled trips and remainders), nonce and alignment; bit-exact with the oracle,
    one sampled warp partial each."""
    rng = np.random.default_rng(2000 + seed)
    for _ in range(6):
        P = int(rng.choice([1, 4]))
        nbytes = 1 << int(rng.integers(4, 21))
        nc = nbytes // (4 * P)
        if nc < 1:
            continue
        choices = [sage.SAGE_AUTO, sage.SAGE_HYBRID, sage.SAGE_GLOBAL]
        if nbytes <= (128 << 10 if P == 1 else 64 << 10):
            choices.append(sage.SAGE_SMEM)
        placement = int(rng.choice(choices))
        blocks = 2 * int(rng.integers(1, 3))
        rounds = int(rng.integers(0, 300))
        nonce = int(rng.integers(0, 2**64, dtype=np.uint64))
        region = make_region(nbytes, fill_seed=int(rng.integers(0, 2**31)))
        d, _keep = to_dev(region, dev, align_offset=32 * int(rng.integers(0, 8)))
        if (d.data_ptr() >> 32) != ((d.data_ptr() + nbytes - 1) >> 32):
            placement = sage.SAGE_AUTO            # the ILP-2 forms need one 4 GiB window
        pw = torch.zeros(blocks * 1024 // 32, dtype=torch.int64, device=dev)
        with sage.Context(blocks=blocks, threads=1024, pick_words=P, placement=placement) as ctx:
            res = ctx.attest_debug(nonce, d, rounds, pw)
        want = oracle.attest(nonce, region, d.data_ptr(), rounds, blocks, 1024, P)
        case = dict(P=P, nbytes=nbytes, placement=placement, used=res.placement, ilp=res.ilp, blocks=blocks,
                    rounds=rounds)
        assert res.checksum == want, case
        if placement == sage.SAGE_HYBRID or (placement == sage.SAGE_SMEM and P == 1):
            assert res.ilp == 2, case
        parts = [int(v) & M64 for v in pw.cpu().tolist()]
        w = int(rng.integers(0, len(parts)))
        assert parts[w] == oracle.warp_sum(nonce, region, d.data_ptr(), rounds, w, P), case


def test_tiny_regions_below_bulk_granule(dev):
    """Nc = 1 and 2 with P = 1 (4- and 8-byte regions) take the non-TMA staging path."""
    for nbytes in (4, 8):
        region = make_region(nbytes, fill_seed=nbytes)
        d, _keep = to_dev(region, dev)
        for placement in (sage.SAGE_SMEM, sage.SAGE_GLOBAL):
            with sage.Context(blocks=2, threads=64, placement=placement) as ctx:
                res = ctx.attest(77, d, 50)
            assert res.checksum == oracle.attest(77, region, d.data_ptr(), 50, 2, 64, 1)


def test_zero_rounds(dev):
    region = make_region(1024)
    d, _keep = to_dev(region, dev)
    with sage.Context(blocks=3, threads=96) as ctx:
        res = ctx.attest(5, d, 0)
    assert res.checksum == oracle.attest(5, region, d.data_ptr(), 0, 3, 96, 1)


@pytest.mark.parametrize("P", [1, 4, 8])
def test_smem_and_global_placements_agree(dev, P):
    region = make_region(4 * P * 2048, prefix=launched_kernel_prefix(4 * P * 2048, blocks=4, threads=256, pick_words=P,
                                                                     placement=sage.SAGE_SMEM))
    d, _keep = to_dev(region, dev)
    out = {}
    for placement in (sage.SAGE_SMEM, sage.SAGE_GLOBAL):
        with sage.Context(blocks=4, threads=256, pick_words=P, placement=placement) as ctx:
            out[placement] = ctx.attest(0xABC, d, 300).checksum
    assert out[sage.SAGE_SMEM] == out[sage.SAGE_GLOBAL] == oracle.attest(0xABC, region, d.data_ptr(), 300, 4, 256, P)


def test_full_occupancy_repeatable_and_sampled(dev):
    """Full occupancy (2 x SMs x 1024), 8 KiB SMEM region: repeat runs are
    bit-identical (atomic-order independence, Q11), the per-warp partials sum
    to the checksum, and sampled warps match the oracle exactly."""
    region = make_region(8192, prefix=launched_kernel_prefix(8192))
    d, _keep = to_dev(region, dev)
    R = 2000
    with sage.Context() as ctx:
        info = ctx.query()
        n = info.blocks * info.threads
        pw = torch.zeros(n // 32, dtype=torch.int64, device=dev)
        r1 = ctx.attest_debug(0x5151, d, R, pw)
        r2 = ctx.attest(0x5151, d, R)
    assert r1.checksum == r2.checksum
    parts = [int(v) & M64 for v in pw.cpu().tolist()]
    assert sum(parts) & M64 == r1.checksum
    rng = np.random.default_rng(4)
    sample = sorted({0, n // 32 - 1, *[int(w) for w in rng.integers(0, n // 32, 6)]})
    for w in sample:
        assert parts[w] == oracle.warp_sum(0x5151, region, d.data_ptr(), R, w, 1), w


def test_bench_config_full_rounds_sampled(dev):
    """configs[1] as bench.py times it: full occupancy, 8 KiB SMEM region,
    10^5 rounds; sum consistency plus 4 sampled warps recomputed by the oracle."""
    region = make_region(8192, prefix=launched_kernel_prefix(8192))
    d, _keep = to_dev(region, dev)
    R = 100_000
    nonce = nonces(1)[0]
    with sage.Context() as ctx:
        info = ctx.query()
        n = info.blocks * info.threads
        pw = torch.zeros(n // 32, dtype=torch.int64, device=dev)
        res = ctx.attest_debug(nonce, d, R, pw)
    parts = [int(v) & M64 for v in pw.cpu().tolist()]
    assert sum(parts) & M64 == res.checksum
    for w in (0, 1, n // 64, n // 32 - 1):
        assert parts[w] == oracle.warp_sum(nonce, region, d.data_ptr(), R, w, 1), w


@pytest.mark.parametrize("P", [1, 4, 8])
def test_hbm_region_sampled(dev, P):
    """configs[2]: 256 MiB region in HBM (GLOBAL placement), sampled warps."""
    nbytes = 256 << 20
    g = torch.Generator(device=dev)
    g.manual_seed(P)
    d = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=dev, generator=g)
    region = d.cpu().numpy()
    R = 10_000                                           # bench.py's c3 round count
    with sage.Context(pick_words=P) as ctx:
        info = ctx.query()
        n = info.blocks * info.threads
        pw = torch.zeros(n // 32, dtype=torch.int64, device=dev)
        res = ctx.attest_debug(99, d, R, pw)
        assert res.placement == sage.SAGE_GLOBAL
    parts = [int(v) & M64 for v in pw.cpu().tolist()]
    assert sum(parts) & M64 == res.checksum
    for w in (0, 12345 % (n // 32), n // 32 - 1):
        assert parts[w] == oracle.warp_sum(99, region, d.data_ptr(), R, w, P), w


@pytest.mark.parametrize("P", [1, 4, 8])
def test_region_straddling_4gib_boundary(dev, P):
    """Chunk data pointers whose high 32 bits differ inside one region (R5/R6 carry)."""
    big = torch.empty((4 << 30) + (1 << 20), dtype=torch.uint8, device=dev)
    base0 = big.data_ptr()
    boundary = ((base0 >> 32) + 1) << 32
    nbytes = 4 * P * 1024
    start = boundary - nbytes // 2 - base0
    d = big[start:start + nbytes]
    region = make_region(nbytes, fill_seed=P)
    d.copy_(torch.from_numpy(region))
    assert (d.data_ptr() >> 32) != ((d.data_ptr() + nbytes - 1) >> 32)
    for placement in (sage.SAGE_SMEM, sage.SAGE_GLOBAL):
        with sage.Context(blocks=2, threads=128, pick_words=P, placement=placement) as ctx:
            res = ctx.attest(31337, d, 200)
        assert res.checksum == oracle.attest(31337, region, d.data_ptr(), 200, 2, 128, P)
    del big


def test_largest_smem_region(dev):
    """64 KiB is the largest region staged into SMEM at 2 CTAs/SM."""
    region = make_region(65536, prefix=launched_kernel_prefix(65536, blocks=3, threads=128))
    d, _keep = to_dev(region, dev)
    with sage.Context(blocks=3, threads=128) as ctx:
        assert ctx.placement_for(65536) == sage.SAGE_SMEM
        assert ctx.placement_for(131072) == sage.SAGE_GLOBAL
        res = ctx.attest(8, d, 100)
    assert res.placement == sage.SAGE_SMEM
    assert res.checksum == oracle.attest(8, region, d.data_ptr(), 100, 3, 128, 1)


def test_async_and_host_forms(dev):
    region = make_region(8192, prefix=launched_kernel_prefix(8192))
    d, _keep = to_dev(region, dev)
    with sage.Context(blocks=2, threads=256) as ctx:
        raw = torch.zeros(4, dtype=torch.int64, device=dev)
        ctx.attest_async(11, d, 123, raw)
        torch.cuda.synchronize()
        dec = sage.decode_raw([int(v) for v in raw.cpu().tolist()])
        assert dec.checksum == ctx.attest(11, d, 123).checksum == oracle.attest(11, region, d.data_ptr(), 123, 2, 256)
        host = torch.from_numpy(region).pin_memory()
        va = ctx.host_region_va(8192)
        res = ctx.attest_host(11, host, 123)
        assert res.region_va == va
        assert res.checksum == oracle.attest(11, region, va, 123, 2, 256)


def test_occupancy_and_registers(dev):
    """Full occupancy: 2048 logical threads per SM and the whole 64 K
    register file allocated -- 2 CTAs x 1024 threads x 32 registers, or (the P=1
    SMEM kernel, ILP 2) 1 CTA x 1024 threads x 2 lane states x 64 allocated registers."""
    for P in (1, 4, 8):
        with sage.Context(pick_words=P) as ctx:
            info = ctx.query()
            assert info.threads == 1024 and info.blocks == 2 * info.sm_count
            assert info.ilp_smem == (2 if P == 1 else 1)
            assert info.ctas_per_sm_smem * info.ilp_smem == 2 and info.ctas_per_sm_global == 2
            # registers are allocated per warp in units of 256 (8 per thread)
            assert info.ctas_per_sm_smem * info.threads * (-(-info.regs_per_thread // 8) * 8) == 65536


def test_ilp2_and_ilp1_kernels_agree(dev):
    """The c2a kernel (ILP 2, one CTA per SM) and the ILP 1 kernel it falls back to
    (odd block count) compute the same SCS-2 result for the same logical threads."""
    region = torch.from_numpy(make_region(8192)).to(dev)
    for blocks in (2, 4):
        with sage.Context(blocks=blocks, threads=1024) as ctx:
            a = ctx.attest(0xC2A, region, 300)
        assert a.ilp == 2
        want = oracle.attest(0xC2A, region.cpu().numpy(), region.data_ptr(), 300, blocks, 1024, 1)
        assert a.checksum == want
    with sage.Context(blocks=3, threads=1024) as ctx:
        b = ctx.attest(0xC2A, region, 300)
    assert b.ilp == 1
    assert b.checksum == oracle.attest(0xC2A, region.cpu().numpy(), region.data_ptr(), 300, 3, 1024, 1)


def test_argument_errors(dev):
    region = torch.zeros(1 << 20, dtype=torch.uint8, device=dev)
    with sage.Context(blocks=1, threads=32) as ctx:
        for nbytes in (0, 12, 24, 3 * 4096):             # empty, not 4P*2^k
            with pytest.raises(sage.SageError) as e:
                ctx.attest(0, region, 1, nbytes=nbytes)
            assert e.value.code == sage.SAGE_EINVAL
        with pytest.raises(sage.SageError) as e:
            ctx.attest(0, region.data_ptr() + 4, 1, nbytes=4096)
        assert e.value.code == sage.SAGE_EINVAL
        with pytest.raises(sage.SageError) as e:
            ctx.attest(0, region, 1 << 32, nbytes=4096)
        assert e.value.code == sage.SAGE_EINVAL
        with pytest.raises(sage.SageError) as e:
            ctx.attest(0, 0, 1, nbytes=4096)
        assert e.value.code == sage.SAGE_EINVAL
    with sage.Context(blocks=1, threads=32, pick_words=8) as ctx:
        with pytest.raises(sage.SageError) as e:
            ctx.attest(0, region.data_ptr() + 16, 1, nbytes=4096)
        assert e.value.code == sage.SAGE_EINVAL
    with sage.Context(blocks=1, threads=32, placement=sage.SAGE_SMEM) as ctx:
        with pytest.raises(sage.SageError) as e:
            ctx.attest(0, region, 1, nbytes=1 << 20)
        assert e.value.code == sage.SAGE_EUNSUPPORTED


def test_host_pointers_rejected_without_faulting(dev):
    """A host buffer where the kernel needs device memory is SAGE_EINVAL (checked
    with cudaPointerGetAttributes), not an illegal-address fault that would leave
    the CUDA context unusable; the context keeps working afterwards.  Pinned host
    memory is device-mapped under UVA and is accepted."""
    buf = np.zeros(4096 + 64, dtype=np.uint8)
    plain = buf.ctypes.data + (-buf.ctypes.data % 64)          # 64-B aligned, unregistered host memory
    region = torch.zeros(4096, dtype=torch.uint8, device=dev)
    with sage.Context(blocks=1, threads=32) as ctx:
        before = ctx.attest(7, region, 100).checksum
        with pytest.raises(sage.SageError) as e:
            ctx.attest(7, plain, 100, nbytes=4096)
        assert e.value.code == sage.SAGE_EINVAL and "host memory" in str(e.value)
        with pytest.raises(sage.SageError) as e:
            ctx.attest_async(7, region, 100, plain)
        assert e.value.code == sage.SAGE_EINVAL
        with pytest.raises(sage.SageError) as e:
            ctx.attest_debug(7, region, 100, plain)
        assert e.value.code == sage.SAGE_EINVAL
        with pytest.raises(sage.SageError) as e:
            ctx.attest_coverage(7, region, 100, plain)
        assert e.value.code == sage.SAGE_EINVAL
        with pytest.raises(sage.SageError) as e:
            ctx.kernel_hash(b"r", plain, nbytes=64)
        assert e.value.code == sage.SAGE_EINVAL
        pinned = torch.zeros(4096, dtype=torch.uint8).pin_memory()
        res = ctx.attest(7, pinned, 100)
        assert res.region_va == pinned.data_ptr()
        assert ctx.attest(7, region, 100).checksum == before


def test_maximum_chunk_count(dev):
    """Nc = 2^32 (the SCS-1 maximum): a 16 GiB P=1 region, mask 0xFFFFFFFF,
    64-bit chunk offsets.  Zero-filled except one marker word per 64 MiB on both
    sides (the host copy is a lazily-allocated numpy zeros array)."""
    import numpy as np
    nbytes = 1 << 34
    try:
        d = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    except RuntimeError:
        pytest.skip("not enough device memory")
    host = np.zeros(nbytes, dtype=np.uint8)
    for k in range(0, nbytes, 64 << 20):
        host[k:k + 4] = np.frombuffer((k // (64 << 20) + 1).to_bytes(4, "little"), dtype=np.uint8)
        d[k:k + 4] = torch.from_numpy(host[k:k + 4].copy()).to(dev)
    with sage.Context(blocks=2, threads=64) as ctx:
        res = ctx.attest(0xBEEF, d, 300)
        assert res.placement == sage.SAGE_GLOBAL
    assert res.checksum == oracle.attest(0xBEEF, host, d.data_ptr(), 300, 2, 64, 1)
    del d


def test_multiple_waves(dev):
    """More CTAs than fit at once (3 x SMs x 1024 threads): the result is the
    same function of the linear thread index."""
    region = make_region(4096, fill_seed=9)
    d, _keep = to_dev(region, dev)
    with sage.Context(blocks=1, threads=32) as c0:
        sms = c0.query().sm_count
    blocks = 3 * sms
    pw = torch.zeros(blocks * 1024 // 32, dtype=torch.int64, device=dev)
    with sage.Context(blocks=blocks, threads=1024) as ctx:
        res = ctx.attest_debug(21, d, 40, pw)
    parts = [int(v) & M64 for v in pw.cpu().tolist()]
    assert sum(parts) & M64 == res.checksum
    for w in (0, len(parts) // 2, len(parts) - 1):
        assert parts[w] == oracle.warp_sum(21, region, d.data_ptr(), 40, w, 1)


def test_p8_auto_placement_is_global(dev):
    region = make_region(8192, prefix=launched_kernel_prefix(8192, blocks=2, threads=96, pick_words=8))
    d, _keep = to_dev(region, dev)
    with sage.Context(blocks=2, threads=96, pick_words=8) as ctx:
        assert ctx.placement_for(8192) == sage.SAGE_GLOBAL
        res = ctx.attest(0x88, d, 250)
    assert res.checksum == oracle.attest(0x88, region, d.data_ptr(), 250, 2, 96, 8)


def test_async_attestation_in_cuda_graph(dev):
    """sage_attest_async is capturable: a CUDA graph of zero-fill + attestation,
    replayed twice, reproduces the synchronous checksum."""
    region = make_region(8192, prefix=launched_kernel_prefix(8192))
    d, _keep = to_dev(region, dev)
    s = torch.cuda.Stream()
    raw = torch.zeros(4, dtype=torch.int64, device=dev)
    with sage.Context(blocks=4, threads=256, stream=s) as ctx:
        ctx.attest(1, d, 10)                                  # warm the kernel / attributes outside capture
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            raw.zero_()
            ctx.attest_async(0x6A, d, 500, raw)
        for _ in range(2):
            g.replay()
            s.synchronize()
            got = sage.decode_raw([int(v) for v in raw.cpu().tolist()]).checksum
            assert got == oracle.attest(0x6A, region, d.data_ptr(), 500, 4, 256, 1)


def test_two_contexts_on_concurrent_streams(dev):
    """Independent contexts on their own streams (e.g. two verifier sessions)
    give the same results as serial runs."""
    import threading
    region = make_region(4096, fill_seed=77)
    d, _keep = to_dev(region, dev)
    want = {n: oracle.attest(n, region, d.data_ptr(), 300, 2, 128, 1) for n in (101, 202)}
    got = {}

    def run(n):
        with sage.Context(blocks=2, threads=128) as ctx:
            got[n] = ctx.attest(n, d, 300).checksum

    ts = [threading.Thread(target=run, args=(n,)) for n in want]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert got == want


def test_one_context_shared_by_threads(dev):
    """Calls on one context from several threads are serialised by its lock."""
    import threading
    region = make_region(4096, fill_seed=78)
    d, _keep = to_dev(region, dev)
    nonces_ = list(range(300, 308))
    want = {n: oracle.attest(n, region, d.data_ptr(), 200, 1, 64, 1) for n in nonces_}
    got = {}
    with sage.Context(blocks=1, threads=64) as ctx:
        def run(ns):
            for n in ns:
                got[n] = ctx.attest(n, d, 200).checksum
        ts = [threading.Thread(target=run, args=(nonces_[k::4],)) for k in range(4)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    assert got == want


@pytest.mark.parametrize("P", [4, 8])
def test_full_occupancy_wide_picks_sampled(dev, P):
    """P = 4 (SMEM, 16-B picks) and P = 8 (AUTO -> L1-resident GLOBAL, 32-B picks)
    at full occupancy, 8 KiB region, 10^4 rounds: Σ-consistency + sampled warps."""
    region = make_region(8192, prefix=launched_kernel_prefix(8192, pick_words=P))
    d, _keep = to_dev(region, dev)
    R = 10_000
    with sage.Context(pick_words=P) as ctx:
        info = ctx.query()
        n = info.blocks * info.threads
        pw = torch.zeros(n // 32, dtype=torch.int64, device=dev)
        res = ctx.attest_debug(0xE0 + P, d, R, pw)
        assert res.placement == (sage.SAGE_SMEM if P == 4 else sage.SAGE_GLOBAL)
    parts = [int(v) & M64 for v in pw.cpu().tolist()]
    assert sum(parts) & M64 == res.checksum
    for w in (0, n // 96, n // 32 - 1):
        assert parts[w] == oracle.warp_sum(0xE0 + P, region, d.data_ptr(), R, w, P), w


def test_ilp2_smem_region_up_to_128k(dev):
    """At the ILP-2 geometry (one CTA per SM) SAGE_AUTO stages regions up to 128 KiB in
    shared memory; bit-exact with the oracle and with GLOBAL."""
    region = make_region(128 << 10, prefix=launched_kernel_prefix(128 << 10, blocks=2, threads=1024))
    d, _keep = to_dev(region, dev)
    with sage.Context(blocks=2, threads=1024) as ctx:
        assert ctx.query().smem_region_max == 128 << 10
        assert ctx.placement_for(128 << 10) == sage.SAGE_SMEM
        res = ctx.attest(0x128, d, 200)
    assert res.placement == sage.SAGE_SMEM and res.ilp == 2
    with sage.Context(blocks=2, threads=1024, placement=sage.SAGE_GLOBAL) as ctx:
        glob = ctx.attest(0x128, d, 200)
    assert res.checksum == glob.checksum == oracle.attest(0x128, region, d.data_ptr(), 200, 2, 1024, 1)
    with sage.Context(blocks=2, threads=512, placement=sage.SAGE_SMEM) as ctx:   # ILP 1: 64 KiB at most
        assert ctx.query().smem_region_max == 64 << 10
        with pytest.raises(sage.SageError) as e:
            ctx.attest(0x128, d, 10)
        assert e.value.code == sage.SAGE_EUNSUPPORTED


@pytest.mark.parametrize("nbytes", [256 << 10, 512 << 10, 1 << 20])
def test_hybrid_placement_bit_exact(dev, nbytes):
    """SAGE_HYBRID (first 192 KiB in shared memory, the rest read in place): chosen by
    SAGE_AUTO for 128 KiB < region <= 1 MiB at a 1024-thread, even-block geometry, and
    bit-exact with the oracle and with the GLOBAL placement."""
    region = make_region(nbytes, prefix=launched_kernel_prefix(nbytes, blocks=2, threads=1024), fill_seed=nbytes)
    d, _keep = to_dev(region, dev, align_offset=16)
    out = {}
    for placement in (sage.SAGE_AUTO, sage.SAGE_GLOBAL):
        with sage.Context(blocks=2, threads=1024, placement=placement) as ctx:
            res = ctx.attest(0x48B, d, 200)
            out[placement] = res
    assert out[sage.SAGE_AUTO].placement == sage.SAGE_HYBRID and out[sage.SAGE_AUTO].ilp == 2
    assert out[sage.SAGE_GLOBAL].placement == sage.SAGE_GLOBAL
    want = oracle.attest(0x48B, region, d.data_ptr(), 200, 2, 1024, 1)
    assert out[sage.SAGE_AUTO].checksum == out[sage.SAGE_GLOBAL].checksum == want


@pytest.mark.parametrize("nbytes,auto", [(128 << 10, sage.SAGE_GLOBAL), (256 << 10, sage.SAGE_HYBRID),
                                         (512 << 10, sage.SAGE_HYBRID), (1 << 20, sage.SAGE_HYBRID)])
def test_hybrid_p4_bit_exact(dev, nbytes, auto):
    """The P = 4 SAGE_HYBRID form (16-B picks; LDS.128 from the staged 192 KiB,
    LDG.128 in place): SAGE_AUTO takes it from 256 KiB to 1 MiB (GLOBAL at 128 KiB,
    where reading in place is faster); forced, auto and GLOBAL placements are
    bit-exact with the oracle."""
    region = make_region(nbytes, prefix=launched_kernel_prefix(nbytes, blocks=2, threads=1024, pick_words=4),
                         fill_seed=nbytes + 4)
    d, _keep = to_dev(region, dev, align_offset=16)
    out = {}
    for placement in (sage.SAGE_AUTO, sage.SAGE_HYBRID, sage.SAGE_GLOBAL):
        with sage.Context(blocks=2, threads=1024, pick_words=4, placement=placement) as ctx:
            out[placement] = ctx.attest(0x48B4, d, 200)
    assert out[sage.SAGE_AUTO].placement == auto
    assert out[sage.SAGE_HYBRID].placement == sage.SAGE_HYBRID and out[sage.SAGE_HYBRID].ilp == 2
    assert out[sage.SAGE_GLOBAL].placement == sage.SAGE_GLOBAL
    want = oracle.attest(0x48B4, region, d.data_ptr(), 200, 2, 1024, 4)
    assert out[sage.SAGE_AUTO].checksum == out[sage.SAGE_HYBRID].checksum == out[sage.SAGE_GLOBAL].checksum == want


@pytest.mark.parametrize("rounds", [0, 1, 2, 3, 37])
def test_hybrid_p4_forced_small_region(dev, rounds):
    """Forced P = 4 SAGE_HYBRID on a 64 KiB region stages all of it (every pick an
    LDS.128), at the round-loop edge cases; P = 8 has no HYBRID form."""
    region = make_region(64 << 10, fill_seed=4 + rounds)
    d, _keep = to_dev(region, dev)
    with sage.Context(blocks=4, threads=1024, pick_words=4, placement=sage.SAGE_HYBRID) as ctx:
        res = ctx.attest(0x4A + rounds, d, rounds)
    assert res.placement == sage.SAGE_HYBRID and res.ilp == 2
    assert res.checksum == oracle.attest(0x4A + rounds, region, d.data_ptr(), rounds, 4, 1024, 4)
    with sage.Context(blocks=2, threads=1024, pick_words=8, placement=sage.SAGE_HYBRID) as ctx:
        with pytest.raises(sage.SageError) as e:
            ctx.attest(5, d, 10)
        assert e.value.code == sage.SAGE_EUNSUPPORTED
    with sage.Context(blocks=2, threads=1024, pick_words=8) as ctx:
        assert ctx.placement_for(512 << 10) == sage.SAGE_GLOBAL


def test_hybrid_forced_small_region_and_unsupported_geometry(dev):
    """Forced SAGE_HYBRID on an 8 KiB region stages all of it; without its geometry
    (P = 1 or 4, 1024-thread blocks, even block count) it is SAGE_EUNSUPPORTED."""
    region = make_region(8192)
    d, _keep = to_dev(region, dev)
    with sage.Context(blocks=4, threads=1024, placement=sage.SAGE_HYBRID) as ctx:
        res = ctx.attest(5, d, 150)
    assert res.placement == sage.SAGE_HYBRID
    assert res.checksum == oracle.attest(5, region, d.data_ptr(), 150, 4, 1024, 1)
    for kw in ({"blocks": 2, "threads": 512}, {"blocks": 3, "threads": 1024}):
        with sage.Context(placement=sage.SAGE_HYBRID, **kw) as ctx:
            with pytest.raises(sage.SageError) as e:
                ctx.attest(5, d, 10)
            assert e.value.code == sage.SAGE_EUNSUPPORTED
    with sage.Context(blocks=2, threads=1024) as ctx:     # AUTO at other geometries: GLOBAL
        assert ctx.placement_for(128 << 10) == sage.SAGE_SMEM
        assert ctx.placement_for(256 << 10) == sage.SAGE_HYBRID
        assert ctx.placement_for(2 << 20) == sage.SAGE_GLOBAL
    with sage.Context(blocks=3, threads=1024) as ctx:
        assert ctx.placement_for(512 << 10) == sage.SAGE_GLOBAL


@pytest.mark.parametrize("nbytes", [128 << 10, 512 << 10])
def test_ilp2_placements_straddling_region_run_global(dev, nbytes):
    """A region over 64 KiB whose chunk addresses straddle a 4 GiB boundary cannot use
    the ILP-2 kernels' 32-bit data pointer; SAGE_AUTO runs it GLOBAL, bit-exact, and
    forcing SMEM / HYBRID is SAGE_EUNSUPPORTED."""
    big = torch.empty((4 << 30) + (2 << 20), dtype=torch.uint8, device=dev)
    base0 = big.data_ptr()
    boundary = ((base0 >> 32) + 1) << 32
    start = boundary - nbytes // 2 - base0
    d = big[start:start + nbytes]
    region = make_region(nbytes, fill_seed=77)
    d.copy_(torch.from_numpy(region))
    with sage.Context(blocks=2, threads=1024) as ctx:
        res = ctx.attest(77, d, 100)
    assert res.placement == sage.SAGE_GLOBAL
    assert res.checksum == oracle.attest(77, region, d.data_ptr(), 100, 2, 1024, 1)
    forced = sage.SAGE_SMEM if nbytes <= (128 << 10) else sage.SAGE_HYBRID
    with sage.Context(blocks=2, threads=1024, placement=forced) as ctx:
        with pytest.raises(sage.SageError) as e:
            ctx.attest(77, d, 10)
        assert e.value.code == sage.SAGE_EUNSUPPORTED
    del big


@pytest.mark.parametrize("P", [1, 4, 8])
def test_paper_buffer_full_occupancy_sampled(dev, P):
    """c2c / c2cp4 / c2cp8 as bench.py times them: the paper's 524,288-B buffer
     at full occupancy, 10^5 rounds (P = 1, 4, 8); sum
    consistency plus sampled warps.  P = 1 runs SAGE_HYBRID."""
    region = make_region(512 << 10, prefix=launched_kernel_prefix(512 << 10, pick_words=P))
    d, _keep = to_dev(region, dev)
    R = 100_000
    with sage.Context(pick_words=P) as ctx:
        info = ctx.query()
        n = info.blocks * info.threads
        pw = torch.zeros(n // 32, dtype=torch.int64, device=dev)
        res = ctx.attest_debug(0xC2C + P, d, R, pw)
        assert res.placement == ctx.placement_for(512 << 10)
    if P == 1:
        assert res.placement == sage.SAGE_HYBRID
    parts = [int(v) & M64 for v in pw.cpu().tolist()]
    assert sum(parts) & M64 == res.checksum
    for w in (0, 1, n // 64, n // 32 - 1):
        assert parts[w] == oracle.warp_sum(0xC2C + P, region, d.data_ptr(), R, w, P), w


def test_no_other_kernel_runs_beside_an_attestation(dev):
    """Full occupancy leaves no room for another kernel: a tiny kernel
    launched on a second stream right after the attestation cannot start until
    the attestation's CTAs leave their SMs, so it finishes only at the end of the
    attestation; with a half-occupancy grid (control) it runs at once."""
    region = torch.from_numpy(make_region(8192)).to(dev)
    side = torch.zeros(1024, device=dev)
    sa, sb = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    for blocks, threads, full in ((0, 0, True), (148, 512, False)):
        with sage.Context(blocks=blocks, threads=threads, stream=sa) as ctx:
            raw = torch.zeros(4, dtype=torch.int64, device=dev)
            ctx.attest_async(1, region, 200, raw)                       # warm-up
            torch.cuda.synchronize(dev)
            raw.zero_()
            e0, e1, eb = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            with torch.cuda.stream(sa):
                e0.record(sa)
                ctx.attest_async(2, region, 20_000, raw)              # ~11 ms at full occupancy
                e1.record(sa)
            with torch.cuda.stream(sb):
                side.add_(1.0)
                eb.record(sb)
            torch.cuda.synchronize(dev)
            t_att, t_side = e0.elapsed_time(e1), e0.elapsed_time(eb)
            print("co-residency probe: blocks=%d threads=%d attestation %.3f ms, side kernel done at %.3f ms"
                  % (blocks, threads, t_att, t_side))
        if full:
            assert t_side > 0.9 * t_att, (t_side, t_att)
        else:
            assert t_side < 0.5 * t_att, (t_side, t_att)


def test_relocated_copy_gives_a_different_checksum(dev):
    """The data pointer is folded in every round, so the same bytes
    attested at another device address (a relocated copy of the verification
    function) give a different checksum -- each equal to the oracle's at its own VA."""
    region = make_region(8192, prefix=launched_kernel_prefix(8192))
    d1, _k1 = to_dev(region, dev)
    d2, _k2 = to_dev(region, dev, align_offset=4096)
    assert d1.data_ptr() != d2.data_ptr()
    with sage.Context(blocks=2, threads=64) as ctx:
        c1 = ctx.attest(C1_NONCE, d1, 500).checksum
        c2 = ctx.attest(C1_NONCE, d2, 500).checksum
    assert c1 != c2
    assert c1 == oracle.attest(C1_NONCE, region, d1.data_ptr(), 500, 2, 64, 1)
    assert c2 == oracle.attest(C1_NONCE, region, d2.data_ptr(), 500, 2, 64, 1)


def test_single_bit_flips_change_the_gpu_checksum(dev):
    """Self-verification: flipping any one bit of the region changes
    the attestation result; 16 random bits of an 8 KiB region at full occupancy
    with enough rounds that every word is read (R = 64), each result equal to
    the oracle's on the flipped bytes."""
    region = make_region(8192, prefix=launched_kernel_prefix(8192))
    d, _keep = to_dev(region, dev)
    rng = np.random.default_rng(11)
    with sage.Context() as ctx:
        base_cs = ctx.attest(0xF11B, d, 64).checksum
        info = ctx.query()
        for bit in rng.integers(0, 8192 * 8, 16):
            flipped = region.copy()
            flipped[bit // 8] ^= np.uint8(1 << (bit % 8))
            d.copy_(torch.from_numpy(flipped))
            cs = ctx.attest(0xF11B, d, 64).checksum
            assert cs != base_cs, int(bit)
            w = int(rng.integers(0, info.blocks * info.threads // 32))
            pw = torch.zeros(info.blocks * info.threads // 32, dtype=torch.int64, device=dev)
            ctx.attest_debug(0xF11B, d, 64, pw)
            assert int(pw[w].item()) & M64 == oracle.warp_sum(0xF11B, flipped, d.data_ptr(), 64, w, 1)
        d.copy_(torch.from_numpy(region))
        assert ctx.attest(0xF11B, d, 64).checksum == base_cs


@pytest.mark.parametrize("rounds", [0, 1, 17, 18, 19, 35, 36, 37, 18 * 7 + 5])
def test_ilp2_round_loop_boundaries(dev, rounds):
    """The c2a kernel runs UNROLL = 18 rounds of both lane states per trip and the
    rest one by one (a10): every trip/remainder split around 0, 1, 18 and 36
    rounds is bit-exact with the oracle (2 CTAs of 1024 threads -> ILP 2)."""
    region = make_region(8192, fill_seed=rounds + 1)
    d, _keep = to_dev(region, dev)
    with sage.Context(blocks=2, threads=1024) as ctx:
        res = ctx.attest(0xB0B + rounds, d, rounds)
    assert res.ilp == 2 and res.placement == sage.SAGE_SMEM
    assert res.checksum == oracle.attest(0xB0B + rounds, region, d.data_ptr(), rounds, 2, 1024, 1)


@pytest.mark.parametrize("rounds", [0, 1, 2, 3, 7])
def test_hybrid_round_loop_boundaries(dev, rounds):
    """SAGE_HYBRID (UNROLL 2 + remainder) at small and odd round counts, region
    256 KiB so 75% of the picks are staged and 25% read in place."""
    region = make_region(256 << 10, fill_seed=rounds + 7)
    d, _keep = to_dev(region, dev)
    with sage.Context(blocks=2, threads=1024) as ctx:
        res = ctx.attest(0x4B + rounds, d, rounds)
    assert res.placement == sage.SAGE_HYBRID and res.ilp == 2
    assert res.checksum == oracle.attest(0x4B + rounds, region, d.data_ptr(), rounds, 2, 1024, 1)


@pytest.mark.parametrize("blocks,threads", [(1, 64), (2, 1024)])
def test_zero_seed_threads(dev, blocks, threads):
    """I2 on the GPU: SplitMix64's only zero output is sm(0), reached by thread g when
    nonce = -(g+1)*G (mod 2^64); that thread's xorshift state must start at G instead
    of 0 (a zero state would stay zero forever).  Nonces that zero the seeds of
    threads 0, 1, 33 and the last one, in the ILP-1 and ILP-2 kernels."""
    G = 0x9E3779B97F4A7C15
    region = make_region(4096, fill_seed=99)
    d, _keep = to_dev(region, dev)
    n = blocks * threads
    with sage.Context(blocks=blocks, threads=threads) as ctx:
        for g in (0, 1, 33, n - 1):
            nonce = (-(g + 1) * G) & M64
            res = ctx.attest(nonce, d, 50)
            assert res.checksum == oracle.attest(nonce, region, d.data_ptr(), 50, blocks, threads, 1), g
