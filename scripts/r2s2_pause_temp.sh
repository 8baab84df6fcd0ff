# Session 2: B200 pause rate vs. time under load / temperature, with NVML polling
# alternated on and off in 30-s windows (12 windows), temperature and power
# logged at 1 Hz throughout.
O=${1:-gpurun_out/pausetemp}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvidia-smi --query-gpu=timestamp,temperature.gpu,temperature.memory,power.draw,clocks.sm,clocks.mem,clocks_event_reasons.active --format=csv -l 1 > $O/temp_1hz.csv 2>&1 &
T=$!
sleep 2
for w in 1 2 3 4 5 6 7 8 9 10 11 12; do
  if [ $((w % 2)) -eq 0 ]; then
    nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv -lms 50 > /dev/null 2>&1 &
    P=$!
  fi
  date +%s.%N > $O/w${w}_start.txt
  timeout 100 python scripts/pause_trace.py --seconds 30 --out $O/w$w.json > $O/w$w.log 2>&1
  if [ $((w % 2)) -eq 0 ]; then kill $P; fi
done
kill $T
