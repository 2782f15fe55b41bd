# d <= 2 sorted-row slice scatter: parity tests, then config 4 / config 2 with and without it
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_determinism.py tests/test_gpu_chunks.py tests/test_gpu_group.py -x -q > gpurun_out/d2_t.log 2>&1; echo "exit $?" >> gpurun_out/d2_t.log
for S in 1 0; do
  GSGPC_SORTED_ROWS=$S timeout 300 python bench.py --config 4 --n 1000000000 --no-e2e --no-cpu --no-cg --steps 3 --warmup 3 > gpurun_out/c4_s$S.json 2> gpurun_out/c4_s$S.err
  GSGPC_SORTED_ROWS=$S timeout 300 python bench.py --config 2 --no-e2e --no-cpu --no-cg --steps 5 --warmup 3 > gpurun_out/c2_s$S.json 2> gpurun_out/c2_s$S.err
done
GSGPC_PROBE_RNG_BPS=8 timeout 200 python tools/precompute_config5_probes.py > gpurun_out/p5_8.json 2>&1
