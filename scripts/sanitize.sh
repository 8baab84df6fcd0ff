# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the small GPU
# parity tests and the SHA-256 kernel tests.  Run on the GPU box from the repo root:
#   bash scripts/sanitize.sh [outdir]
out=${1:-gpurun_out}
mkdir -p "$out"
sel="config1 or random_small or tiny_regions or zero_rounds or placements_agree or straddling or vectors or padding or hybrid_placement or hybrid_forced or hybrid_p4 or ilp2 or host_pointers or boundaries or zero_seed or launched_kernels_code or staging_buffer or owned_stream"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --target-processes all \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_sha256.py tests/test_gpu_boundary.py -m gpu -q -k "$sel" \
    > "$out/sanitizer_$tool.log" 2>&1
  tail -3 "$out/sanitizer_$tool.log" > "$out/sanitizer_$tool.txt"
done
