"""Quick device timing of the checksum kernel over the SURVEY 8(d) configs
(development aid; bench.py is the contract)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2209_03125_b200 import sage  # noqa: E402
from paper_2209_03125_b200.inputs import launched_kernel_prefix, make_region  # noqa: E402


def time_cfg(nbytes, P, R, reps=5, placement=sage.SAGE_AUTO):
    dev = torch.device("cuda:0")
    if nbytes <= (1 << 20):
        region = torch.from_numpy(make_region(nbytes, prefix=launched_kernel_prefix(nbytes, pick_words=P))).to(dev)
    else:
        region = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    with sage.Context(pick_words=P, placement=placement, stream=s.cuda_stream) as ctx:
        info = ctx.query()
        n = info.blocks * info.threads
        raw = torch.zeros(4, dtype=torch.int64, device=dev)
        for _ in range(2):
            raw.zero_()
            ctx.attest_async(1, region, R, raw)
        torch.cuda.synchronize()
        ts = []
        for k in range(reps):
            raw.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            ctx.attest_async(k + 7, region, R, raw)
            e1.record(s)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        dec = sage.decode_raw([int(v) for v in raw.cpu().tolist()])
        t = min(ts)
        rps = n * R / t
        return dict(nbytes=nbytes, P=P, R=R, placement=ctx.placement_for(nbytes), n=n, t_s=t,
                    thread_rounds_per_s=rps, gbps=rps * 4 * P / 1e9, cycles=dec.cycles,
                    device_ns=dec.device_ns, regs=info.regs_per_thread)


if __name__ == "__main__":
    cfgs = [(8192, 1, 100_000), (65536, 1, 100_000), (524288, 1, 20_000), (524288, 4, 20_000),
            (524288, 8, 20_000), (256 << 20, 1, 10_000), (256 << 20, 4, 10_000), (256 << 20, 8, 10_000),
            (8192, 4, 100_000), (8192, 8, 100_000)]
    for c in cfgs:
        print(json.dumps(time_cfg(*c)), flush=True)
