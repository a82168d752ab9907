mkdir -p gpurun_out
timeout 300 python scripts/umma_stage_check.py 2 3 4 > gpurun_out/umma_stage.log 2>&1; echo stage=$?
timeout 300 python scripts/phase_clock.py --n 32 --order 4 --variant 2 > gpurun_out/phase_umma.log 2>&1; echo phase=$?
timeout 600 python scripts/ab_fused.py --n 64 --orders 4 --dtypes float32 --variants 2 > gpurun_out/umma_ab.log 2>&1; echo ab=$?
cat gpurun_out/umma_stage.log | grep rel_all; cat gpurun_out/phase_umma.log gpurun_out/umma_ab.log
