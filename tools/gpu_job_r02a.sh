mkdir -p gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r02a/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02a/gpu_tests.log 2>&1; tail -3 gpurun_out/r02a/gpu_tests.log
timeout 300 python bench.py > gpurun_out/r02a/bench.json 2> gpurun_out/r02a/bench.err; head -c 1500 gpurun_out/r02a/bench.json
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_step2_tb" -s 1 -c 1 -o gpurun_out/r02a/tb_src -f python tools/tb_ncu_target.py bgk > gpurun_out/r02a/ncu.log 2>&1
tail -2 gpurun_out/r02a/ncu.log
