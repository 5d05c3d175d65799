timeout 300 python -m pytest tests/test_gpu_model.py -q -x -p no:cacheprovider -k "reproducible or graph" > gpurun_out/p2.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/p2.log
