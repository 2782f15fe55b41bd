set -x
python bench.py > gpurun_out/r2s_bench_config3.json 2> gpurun_out/r2s_bench_config3.err
python bench.py --config 4 --n 1000000000 --no-cpu --no-e2e --no-cg --steps 5 > gpurun_out/r2s_bench_config4_1e9.json 2>/dev/null
python bench.py --config 5 --no-cpu --no-e2e --steps 5 > gpurun_out/r2s_bench_config5.json 2>/dev/null
python bench.py --config 2 --no-cpu --no-e2e --steps 5 > gpurun_out/r2s_bench_config2.json 2>/dev/null
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2s_launches_config3.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-cg > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_moments_d3c -s 1 -c 1 -o gpurun_out/r2s_k1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-cg > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_efcg_persistent -c 1 -o gpurun_out/r2s_efcg python tools/profile_cg.py 3 40 > gpurun_out/ncu3.log 2>&1
ls -la gpurun_out/*.ncu-rep
