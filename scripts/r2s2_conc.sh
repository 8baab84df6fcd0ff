# Session 2: concurrency sweep of the random-sector gather probe (Little's law)
O=${1:-gpurun_out/conc}
mkdir -p $O
python -c "from bench import microbench; microbench.build()"
for mb in 64 256 2048; do timeout 300 bench/microbench conc $mb >> $O/gather_concurrency.jsonl 2>> $O/conc.err; done
