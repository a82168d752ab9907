mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python scripts/mass_compare.py --n 32 --orders 2 3 4 5 > gpurun_out/mass_compare.jsonl 2> gpurun_out/mass_compare.err; echo mc=$?
cat gpurun_out/mass_compare.jsonl; tail -3 gpurun_out/mass_compare.err
