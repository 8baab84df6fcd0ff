"""Same logical grid (303,104 threads) launched as 1024/512/256/128-thread CTAs:
the checksum must be identical (it depends on n only) and 1024-thread CTAs are
fastest (dev aid)."""
import torch, time, sys
sys.path.insert(0, '.')
from paper_2209_03125_b200 import sage
from paper_2209_03125_b200.inputs import make_region, launched_kernel_prefix
region = torch.from_numpy(make_region(8192, prefix=launched_kernel_prefix(8192))).to('cuda')
s = torch.cuda.Stream()
for threads in (1024, 512, 256, 128):
    blocks = 303104 // threads
    with sage.Context(blocks=blocks, threads=threads, stream=s) as ctx:
        raw = torch.zeros(4, dtype=torch.int64, device='cuda')
        for _ in range(2):
            raw.zero_(); ctx.attest_async(7, region, 100000, raw)
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            raw.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s); ctx.attest_async(7, region, 100000, raw); e1.record(s); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        cs = sage.decode_raw([int(v) for v in raw.cpu().tolist()]).checksum
        print(threads, blocks, min(ts), hex(cs))
