"""Boundary behaviour on the GPU: which kernel an attestation
launches (so the region can carry that kernel's own code),
validation before the host-region staging buffer is touched, stream ordering
of the context-owned stream, and the caller's current device."""
import pytest

torch = pytest.importorskip("torch")

import oracle                                                     # noqa: E402
from paper_2209_03125_b200 import sage                            # noqa: E402
from paper_2209_03125_b200.inputs import kernel_code_prefix, kernel_text, make_region  # noqa: E402

pytestmark = pytest.mark.gpu

# product template sage_checksum_kernel<P, SMEM, STRADDLE, XS, UNROLL, ADDR, COUNT, ILP, PAD>
C2A = "_ZN4sage20sage_checksum_kernelILi1ELb1ELb0ELi16ELi18ELi4ELb0ELi2ELi7EEEvNS_10KernelArgsE"
HYBRID = "_ZN4sage20sage_checksum_kernelILi1ELb1ELb0ELi16ELi2ELi8ELb0ELi2ELi8EEEvNS_10KernelArgsE"
HYBRID_P4 = "_ZN4sage20sage_checksum_kernelILi4ELb1ELb0ELi16ELi1ELi8ELb0ELi2ELi0EEEvNS_10KernelArgsE"
GLOBAL_P1 = "_ZN4sage20sage_checksum_kernelILi1ELb0ELb1ELi16ELi16ELi0ELb0ELi1ELi0EEEvNS_10KernelArgsE"
GLOBAL_P8 = "_ZN4sage20sage_checksum_kernelILi8ELb0ELb1ELi16ELi1ELi0ELb0ELi1ELi0EEEvNS_10KernelArgsE"
SMEM_ILP1 = "_ZN4sage20sage_checksum_kernelILi1ELb1ELb0ELi16ELi32ELi4ELb0ELi1ELi0EEEvNS_10KernelArgsE"


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2209_03125_b200 import build
    build.build()
    return torch.device("cuda:0")


@pytest.mark.parametrize("cfg,nbytes,symbol,placement,ilp", [
    ({}, 8192, C2A, sage.SAGE_SMEM, 2),                       # c2a (bench default)
    ({}, 512 << 10, HYBRID, sage.SAGE_HYBRID, 2),             # c2c, the paper's buffer
    ({"pick_words": 4}, 512 << 10, HYBRID_P4, sage.SAGE_HYBRID, 2),   # c2cp4
    ({}, 256 << 20, GLOBAL_P1, sage.SAGE_GLOBAL, 1),          # c3
    ({"pick_words": 8}, 256 << 20, GLOBAL_P8, sage.SAGE_GLOBAL, 1),
    ({"blocks": 2, "threads": 64}, 4096, SMEM_ILP1, sage.SAGE_SMEM, 1),   # smoke()
])
def test_region_prefix_is_the_launched_kernels_code(dev, cfg, nbytes, symbol, placement, ilp):
    """sage_kernel_symbol names the instantiation the launch uses; the region
    prefix is that kernel's .text (non-empty machine code from the cubin built with
    the library), and the attestation reports the same placement and lane states."""
    with sage.Context(**cfg) as ctx:
        assert ctx.kernel_symbol(nbytes) == symbol
        code = kernel_code_prefix(ctx, nbytes)
        assert len(code) > 4096 and code == kernel_text(symbol)
        assert code[:16] != bytes(16)
        if nbytes <= (1 << 20):
            region = make_region(nbytes, prefix=code)
            d = torch.from_numpy(region).to(dev)
            res = ctx.attest(0x5E1F, d, 20)
            assert (res.placement, res.ilp) == (placement, ilp)
            assert ctx.kernel_symbol(nbytes, d.data_ptr()) == symbol
            n = res.blocks * res.threads
            if n <= 4096:
                assert res.checksum == oracle.attest(0x5E1F, region, d.data_ptr(), 20, res.blocks, res.threads,
                                                     cfg.get("pick_words", 1))


def test_kernel_symbol_rejects_bad_sizes(dev):
    with sage.Context() as ctx:
        for bad in (0, 12, 3 * 4096):
            with pytest.raises(sage.SageError) as e:
                ctx.kernel_symbol(bad)
            assert e.value.code == sage.SAGE_EINVAL


def test_invalid_host_attestation_keeps_the_staging_buffer(dev):
    """sage_attest_host validates region_bytes and rounds before it (re)allocates the
    staging buffer, so a verifier's precomputed VA (sage_host_region_va) survives a
    bogus call, which returns SAGE_EINVAL (not SAGE_ENOMEM)."""
    host = make_region(8192).copy()
    with sage.Context(blocks=2, threads=64) as ctx:
        va = ctx.host_region_va(8192)
        for nbytes, rounds in ((12, 10), (3 << 40, 10), (8192, 1 << 32), (0, 10)):
            with pytest.raises(sage.SageError) as e:
                ctx.attest_host(1, host, rounds, nbytes=nbytes)
            assert e.value.code == sage.SAGE_EINVAL, (nbytes, rounds)
        assert ctx.host_region_va(8192) == va
        res = ctx.attest_host(7, host, 100)
        assert res.region_va == va
        assert res.checksum == oracle.attest(7, host, va, 100, 2, 64, 1)


def test_owned_stream_is_ordered_with_the_default_stream(dev):
    """With no stream configured the context launches on a blocking stream: a region
    rewritten on the legacy default stream behind a ~50 ms spin kernel is fully
    written when the attestation (issued right after, no host sync) reads it."""
    old = make_region(8192, fill_seed=1)
    new = make_region(8192, fill_seed=2)
    d = torch.from_numpy(old).to(dev)
    new_host = torch.from_numpy(new).pin_memory()
    torch.cuda.synchronize()
    assert torch.cuda.current_stream().cuda_stream == 0
    with sage.Context(blocks=2, threads=64) as ctx:
        torch.cuda._sleep(100_000_000)                      # default stream busy ~50 ms
        d.copy_(new_host, non_blocking=True)                # then the region is rewritten
        res = ctx.attest(0xD00D, d, 200)                    # owned stream, no host sync before
    assert res.checksum == oracle.attest(0xD00D, new, d.data_ptr(), 200, 2, 64, 1)


def test_callers_current_device_is_restored(dev):
    """Every entry point restores the caller's current device (single-GPU boxes: the
    device stays the one the caller set, also after init/attest/query/destroy)."""
    torch.cuda.set_device(0)
    region = torch.from_numpy(make_region(4096)).to(dev)
    with sage.Context(device=0, blocks=1, threads=32) as ctx:
        ctx.attest(1, region, 10)
        ctx.query()
        ctx.kernel_symbol(4096)
    assert torch.cuda.current_device() == 0


def test_timing_fields_are_consistent(dev):
    """a13: the device span (%globaltimer, first CTA start -> last
    CTA end) lies inside the host's t1 - t0 and agrees with CUDA events around the
    same launch; max CTA cycles / device span is an SM clock (0.8-2.1 GHz); the
    host overhead around the kernel (launch, 32-B readback) is well under a ms."""
    region = make_region(8192)
    d = torch.from_numpy(region).to(dev)
    s = torch.cuda.Stream()
    raw = torch.zeros(4, dtype=torch.int64, device=dev)
    with sage.Context(stream=s) as ctx:
        for _ in range(2):
            res = ctx.attest(0x7117, d, 20_000)
        assert 0 < res.device_ns <= res.elapsed_ns
        assert res.elapsed_ns - res.device_ns < 1_000_000
        ghz = res.cycles / res.device_ns
        assert 0.8 < ghz < 2.1, ghz
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            raw.zero_()
            e0.record(s)
            ctx.attest_async(0x7117, d, 20_000, raw)
            e1.record(s)
        s.synchronize()
        dec = sage.decode_raw(raw.cpu().tolist())
        ev_ns = e0.elapsed_time(e1) * 1e6
    assert dec.checksum == res.checksum
    assert abs(dec.device_ns - ev_ns) < 0.02 * ev_ns, (dec.device_ns, ev_ns)


def test_device_uuid_names_the_attested_gpu(dev):
    """sage_device_uuid returns the attested GPU's UUID (the id a verifier binds its
    timing model to, verifier.bind_device), the one nvidia-smi reports for the same
    device, and it is stable across contexts."""
    import re
    import subprocess
    with sage.Context() as ctx:
        u = ctx.device_uuid()
    assert re.fullmatch(r"GPU-[0-9a-f]{8}-[0-9a-f]{4}-[0-9a-f]{4}-[0-9a-f]{4}-[0-9a-f]{12}", u), u
    assert u != "GPU-00000000-0000-0000-0000-000000000000"
    with sage.Context(blocks=2, threads=64) as ctx:
        assert ctx.device_uuid() == u
    try:
        smi = subprocess.run(["nvidia-smi", "--query-gpu=uuid", "--format=csv,noheader"], capture_output=True,
                             text=True, timeout=60).stdout.split()
    except (OSError, subprocess.SubprocessError):
        smi = []
    if smi:
        assert u in smi, (u, smi)
