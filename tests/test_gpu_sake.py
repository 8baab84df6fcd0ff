"""SAKE with the device role on the GPU: the checksum c is
the sm_100a attestation kernel and the device hash chain w0..w2 (and H(v1),
H(v0)) is the GPU SHA-256 kernel; the verifier (host) checks them with its own
SHA-256 and the oracle's expected checksum."""
import pytest

torch = pytest.importorskip("torch")

import oracle                                              # noqa: E402
from paper_2209_03125_b200 import sage, sake               # noqa: E402
from paper_2209_03125_b200.inputs import make_region       # noqa: E402

pytestmark = pytest.mark.gpu


def test_key_agreement_with_gpu_device():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    region_np = make_region(4096, fill_seed=21)
    region = torch.from_numpy(region_np).to("cuda")
    R = 500
    with sage.Context(blocks=2, threads=64) as ctx:
        dev = sake.gpu_device_session(ctx, region, R)
        ver = sake.VerifierSession(group=sake.MODP2048, threshold_s=5.0,
                                   expected_checksum=lambda n: oracle.attest(n, region_np, region.data_ptr(), R, 2, 64))
        sk_v, sk_d = sake.run_protocol(ver, dev)
    assert sk_v == sk_d and sk_v > 1
    assert ver.state == dev.state == "done"
