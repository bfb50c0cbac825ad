set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/r2a_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_pytest.log
timeout 300 python tools/kbench.py c2 20 > gpurun_out/r2a_kbench.log 2>&1
FXG_LIB= timeout 300 python tools/kbench.py c3 10 >> gpurun_out/r2a_kbench.log 2>&1
tail -5 gpurun_out/r2a_pytest.log; cat gpurun_out/r2a_kbench.log
