cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1
echo "exit $?" >> gpurun_out/gpu_tests.log
tail -5 gpurun_out/gpu_tests.log
