"""Memory-region inclusion experiment on the GPU:
with N uniform pseudo-random picks over S words, the fraction of words never
read is (1 - 1/S)^N.  The paper evaluates (1 - 1/524288)^100000 and prints
0.082; the formula gives 0.8264 (Q15).  Here the instrumented kernel
(sage_attest_coverage) counts the reads of a real attestation."""
import pytest

torch = pytest.importorskip("torch")

from paper_2209_03125_b200 import sage, verifier          # noqa: E402
from paper_2209_03125_b200.inputs import make_region       # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2209_03125_b200 import build
    build.build()
    return torch.device("cuda:0")


@pytest.mark.parametrize("words", [524288, 131072])
def test_unread_fraction_matches_inclusion_formula(dev, words):
    N = 100_000                                   # picks
    threads, rounds = 32, N // 32 + (1 if N % 32 else 0)
    N = threads * rounds
    region = torch.from_numpy(make_region(4 * words, fill_seed=words)).to(dev)
    counts = torch.zeros(words, dtype=torch.int32, device=dev)
    with sage.Context(blocks=1, threads=threads) as ctx:
        res = ctx.attest_coverage(0xC0FFEE, region, rounds, counts)
        plain = ctx.attest(0xC0FFEE, region, rounds)
    assert res.checksum == plain.checksum             # instrumentation does not change the result
    c = counts.cpu()
    assert int(c.sum()) == N
    unread = float((c == 0).float().mean())
    p = verifier.inclusion_probability(words, N)
    se = (p * (1 - p) / words) ** 0.5
    assert abs(unread - p) < 6 * se + 1e-4, (unread, p)


def test_full_grid_reads_every_word(dev):
    """At full occupancy even a handful of rounds reads every word of the
    paper-sized buffer: 303,104 threads x 16 rounds = 4.8e6 picks over 131,072
    words leaves each unread with probability e^-37."""
    words = 131072
    region = torch.from_numpy(make_region(4 * words, fill_seed=3)).to(dev)
    counts = torch.zeros(words, dtype=torch.int32, device=dev)
    with sage.Context() as ctx:
        info = ctx.query()
        res = ctx.attest_coverage(7, region, 16, counts)
        assert res.checksum == ctx.attest(7, region, 16).checksum
    c = counts.cpu()
    assert int(c.sum()) == info.blocks * info.threads * 16
    assert int((c == 0).sum()) == 0
