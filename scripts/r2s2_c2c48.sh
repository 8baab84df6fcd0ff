# Round 2, session 2: the paper buffer (and its neighbours) at P = 4 / 8 -- GLOBAL
# (product) vs ILP-2 GLOBAL vs the hybrid with FMA-pipe addressing (lab ADDR 10).
O=${1:-gpurun_out/c2c48}
mkdir -p $O
B=bench/variants_c2c48
for pass in 1 2; do
  for b in 524288 262144 1048576; do
    R=100000; [ $b = 1048576 ] && R=20000
    timeout 600 $B $R $b -1 >> $O/c2c48_$b.jsonl 2>> $O/c2c48.err
  done
done
