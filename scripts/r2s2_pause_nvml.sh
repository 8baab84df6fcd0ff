# Session 2: does NVML polling change B200's pause rate?  pause_trace.py (60 s of
# R = 1e4 attestations) alone, beside an `nvidia-smi -lms 50` poller, and beside a
# tight pynvml loop (clocks + power + utilization), alone again at the end.
O=${1:-gpurun_out/pausenvml}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvidia-smi -q > $O/smi_q.txt 2>&1
ps aux > $O/ps.txt 2>&1
timeout 200 python scripts/pause_trace.py --seconds 60 --out $O/alone1.json > $O/alone1.log 2>&1
nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv -lms 50 > /dev/null 2>&1 &
P=$!
timeout 200 python scripts/pause_trace.py --seconds 60 --out $O/smi50.json > $O/smi50.log 2>&1
kill $P
python - > $O/nvml_loop.log 2>&1 <<'PY' &
import time, pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0); n = 0; t = time.time()
while time.time() - t < 75:
    pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM); pynvml.nvmlDeviceGetPowerUsage(h)
    pynvml.nvmlDeviceGetUtilizationRates(h); n += 1
print({"queries": n, "seconds": time.time() - t})
PY
P=$!
sleep 2
timeout 200 python scripts/pause_trace.py --seconds 60 --out $O/nvmlloop.json > $O/nvmlloop.log 2>&1
wait $P
timeout 200 python scripts/pause_trace.py --seconds 60 --out $O/alone2.json > $O/alone2.log 2>&1
