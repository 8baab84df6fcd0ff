"""The replica plumbing on the NCCL backend bench.py uses when every rank owns a
GPU (8(e)): one process on the box's GPU, world size 1 (the pool gives one GPU;
NCCL refuses two ranks on one device).  It runs a real attestation through
libsage.so, then the max-over-ranks timing (all_reduce of a CUDA tensor) and the
gather of the replica record to rank 0 (gather_object) over an initialised NCCL
process group, and checks the record against the oracle."""
import os
import socket

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_nccl_plumbing_world_size_one():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.distributed as dist

    import oracle
    from paper_2209_03125_b200 import build, replicas, sage
    from paper_2209_03125_b200.inputs import make_region
    build.build()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        assert dist.get_backend() == "nccl"
        region = make_region(4096)
        d = torch.from_numpy(region).to(dev)
        nonce = replicas.replica_nonces(0, 1)[0]
        with sage.Context(blocks=1, threads=32) as ctx:
            res = ctx.attest(nonce, d, 500)
            uuid = ctx.device_uuid()
        rec = {"rank": 0, "nonce": nonce, "checksum": "0x%016x" % res.checksum, "device": uuid}
        tmax = replicas.max_over_ranks(res.device_ns * 1e-9, dev)
        allr = replicas.gather_results(rec)
        assert tmax == pytest.approx(res.device_ns * 1e-9)
        assert allr == [rec]
        ok = replicas.verify_replicas(allr, {0: oracle.attest(nonce, region, d.data_ptr(), 500, 1, 32)})
        assert ok == {0: True}
    finally:
        dist.destroy_process_group()
