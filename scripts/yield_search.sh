# Hill-climb over the c2a loop's yield hints on the GPU box (lab; scripts/yield_search.py).
O=${O:-gpurun_out/r2s3_ys}
mkdir -p $O
G=${G:-15}
for g in $(seq 1 $G); do
  python scripts/yield_search.py --state $O/state.json --gen $g --out $O/cand.json --init "13904,14256,14352,15120,15344,15392,15536,16000,16272,17136,17360,17680,18176,18208,18464,18608,19168,19520,19696,20064,20368,20416,21152,21264,21744,23824,24608,25296,25312,25568,26032,26784,26928,27344,27520,27552,28016,28400,28624,28976,29008,29296,30080,30656,30816,30976,31392,31936,32080,32608,34576,35152,35376,35456,35872,35920,37056,37328,38736,38816,39072,39168,39712,39872,40016,40176,40480,40704,40976,41072,41152,41504,41536,41856,42336,42432,42976,43248,43936,43952,44096,45184,45344,45360,45584,46304,46608" --n 30 --k ${K:-10} --margin ${MARGIN:-0.001}
  timeout 300 python scripts/sass_ctl_probe.py --reps 3 --modes orig --flipsets $O/cand.json --out $O/res_$g.jsonl > $O/probe_$g.log 2>&1 || break
  python scripts/yield_search.py --state $O/state.json --update $O/res_$g.jsonl --margin ${MARGIN:-0.001} >> $O/history.jsonl
done
