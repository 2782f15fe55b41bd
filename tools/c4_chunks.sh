for L in 27 28 29 30; do
  GSGPC_DEV_CHUNK_LOG2=$L timeout 300 python bench.py --config 4 --n 1000000000 --no-e2e --no-cpu --no-cg --steps 3 --warmup 3 > gpurun_out/c4_$L.json 2> gpurun_out/c4_$L.err
done
