cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_vcycle.py -x -q -p no:cacheprovider > gpurun_out/t_tr.log 2>&1; echo "rc=$?" >> gpurun_out/t_tr.log
python tools/transfer_bench.py > gpurun_out/transfer_flat.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench3.log 2>&1
python tools/configs_bench.py C1 C3-GS C4 > gpurun_out/configs3.log 2>&1
