# tcgen05 bring-up on the GPU box: primitives, stage parity, A/B timing
mkdir -p gpurun_out
timeout 300 python scripts/umma_check.py > gpurun_out/umma_check.log 2>&1; echo umma_check=$?
timeout 300 python scripts/umma_stage_check.py 2 3 4 > gpurun_out/umma_stage.log 2>&1; echo umma_stage=$?
timeout 600 python scripts/ab_fused.py --n 64 --orders 4 --dtypes float32 --variants 1 2 > gpurun_out/umma_ab.log 2>&1; echo ab=$?
tail -5 gpurun_out/umma_check.log gpurun_out/umma_stage.log gpurun_out/umma_ab.log
