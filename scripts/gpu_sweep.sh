# config 3 degree sweep (fp32 + fp64) and config 5 single GPU, with the default kernels
mkdir -p gpurun_out
timeout 1500 python scripts/sweep.py > gpurun_out/sweep_c3.jsonl 2> gpurun_out/sweep_c3.err; echo sweep=$?
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5=$?
tail -3 gpurun_out/sweep_c3.jsonl; cat gpurun_out/bench_c5.json
