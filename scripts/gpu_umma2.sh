mkdir -p gpurun_out
timeout 300 python scripts/phase_clock.py --n 32 --order 4 --variant 2 > gpurun_out/phase_umma.log 2>&1; echo phase=$?
timeout 300 python scripts/phase_clock.py --n 32 --order 4 --variant 1 >> gpurun_out/phase_umma.log 2>&1; echo phase=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stage_umma -s 2 -c 1 -o gpurun_out/prof_umma python scripts/ab_fused.py --n 32 --orders 4 --dtypes float32 --variants 2 > gpurun_out/ncu_umma.log 2>&1; echo ncu=$?
cat gpurun_out/phase_umma.log
