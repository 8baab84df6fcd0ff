"""GPU kernel hash h = SHA-256(r || code) (SAGE Eq. (9)) against the
pinned C oracle, byte-exact: FIPS vectors split across r and code, padding
boundaries, the SPEC example, and a 1 MiB code region."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle                                      # noqa: E402
from paper_2209_03125_b200 import sage             # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2209_03125_b200 import build
    build.build()
    c = sage.Context(blocks=1, threads=32)
    yield c
    c.close()


def dev_bytes(b):
    t = torch.empty(max(1, len(b)), dtype=torch.uint8, device="cuda")
    if b:
        t[: len(b)].copy_(torch.frombuffer(bytearray(b), dtype=torch.uint8))
    return t


def test_vectors(ctx):
    cases = [(b"", b"abc"), (b"ab", b"c"), (b"abc", b""), (bytes(32), b""),
             (b"abcdbcdecdefdefgefghfghighijhijkijkl", b"mklmnlmnomnopnopq")]
    for r, code in cases:
        h, ns = ctx.kernel_hash(r, dev_bytes(code), nbytes=len(code))
        assert h == oracle.sha256(r, code), (r, code)
        assert ns > 0
    h, _ = ctx.kernel_hash(bytes(32), None)
    assert h.hex() == "66687aadf862bd776c8fc18b8e9f8e20089714856ee233b3902a591d0d5f2925"


def test_padding_boundaries_and_lengths(ctx):
    rng = np.random.default_rng(9)
    for n in list(range(0, 140)) + [447, 448, 2047, 2048, 2049, 4096 + 55, 64 * 32 * 3 + 7]:
        rl = int(rng.integers(0, min(n, 128) + 1))
        m = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        r, code = m[:rl], m[rl:]
        h, _ = ctx.kernel_hash(r, dev_bytes(code), nbytes=len(code))
        assert h == oracle.sha256(r, code), n


def test_large_code_region(ctx):
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    code = torch.randint(0, 256, (1 << 20,), dtype=torch.uint8, device="cuda", generator=g)
    r = bytes(range(32))
    h, ns = ctx.kernel_hash(r, code)
    assert h == oracle.sha256(r, code.cpu().numpy())
    # any single-bit flip in code changes h
    code[12345] ^= 1
    assert ctx.kernel_hash(r, code)[0] != h


def test_errors(ctx):
    with pytest.raises(sage.SageError) as e:
        ctx.kernel_hash(bytes(129), None)
    assert e.value.code == sage.SAGE_EINVAL
