set -x
mkdir -p gpurun_out
python -c "import torch;print(torch.cuda.get_device_name())"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench_rc=$?
timeout 300 python scripts/fma_peak.py > gpurun_out/fma_peak.json 2>&1
CMD="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stage -s 3 -c 1 -o gpurun_out/prof_tc $CMD > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
