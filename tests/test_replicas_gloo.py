"""Multi-process (world_size 2, gloo, CPU) test of the replica plumbing:
independent nonces per rank, result gather to rank 0 only (each record carrying
that rank's own clock sampler summary), max-over-ranks timing, and the rank-0
verification of every replica.  The per-rank checksum comes
from the oracle here (no GPU); on the box it comes from libsage.so."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, outq):
    import numpy as np
    import torch.distributed as dist

    import oracle
    from bench.clocks import ClockSampler
    from paper_2209_03125_b200 import replicas
    from paper_2209_03125_b200.inputs import make_region

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        nonce = replicas.replica_nonces(rank, 1)[0]
        region = make_region(1024)
        base = 0x7F00_0000_0000 + rank * 0x1000
        cs = oracle.attest(nonce, region, base, 50, 1, 32)
        sampler = ClockSampler(rank).start()           # each rank samples its own GPU
        clocks = sampler.stop()
        rec = {"rank": rank, "nonce": nonce, "checksum": "0x%016x" % cs, "device_ns": 1000 + 500 * rank,
               "clocks": clocks}
        allr = replicas.gather_results(rec)
        tmax = replicas.max_over_ranks(1.0 + rank)
        if rank == 0:
            expected = {r["rank"]: oracle.attest(r["nonce"], region, 0x7F00_0000_0000 + r["rank"] * 0x1000, 50, 1, 32)
                        for r in allr}
            ok = replicas.verify_replicas(allr, expected)
            outq.put({"records": allr, "tmax": tmax, "ok": ok})
        else:
            assert tmax == 2.0
            assert allr is None                          # gathered to rank 0 only
        assert np.isfinite(tmax)
    finally:
        dist.destroy_process_group()


def test_two_replicas_gather_and_verify():
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert [r["rank"] for r in res["records"]] == [0, 1]
    assert res["records"][0]["nonce"] != res["records"][1]["nonce"]
    assert res["records"][0]["checksum"] != res["records"][1]["checksum"]
    assert res["tmax"] == 2.0
    assert res["ok"] == {0: True, 1: True}
    # every replica's record carries its own GPU's clock record
    assert [r["clocks"]["gpu"] for r in res["records"]] == [0, 1]
    assert all({"sm_mhz", "sm_max_mhz", "reasons", "samples"} <= set(r["clocks"]) for r in res["records"])


def test_single_process_fallbacks():
    from paper_2209_03125_b200 import replicas
    assert replicas.world() == (1, 0)
    assert replicas.max_over_ranks(3.5) == 3.5
    assert replicas.gather_results({"rank": 0}) == [{"rank": 0}]
    a, b = replicas.replica_nonces(0, 4), replicas.replica_nonces(1, 4)
    assert not set(a) & set(b)


if __name__ == "__main__":
    pytest.main([__file__])
