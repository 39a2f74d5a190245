cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_sai.py tests/test_gpu_vcycle.py -x -q -p no:cacheprovider > gpurun_out/t_tv.log 2>&1; echo "rc=$?" >> gpurun_out/t_tv.log
python bench.py --no-cpu-baseline > gpurun_out/bench_tv.log 2>&1
LDGMG_TVIEW=0 python bench.py --no-cpu-baseline > gpurun_out/bench_tv0.log 2>&1
python tools/configs_bench.py C5 C3-SAI C4 --c5n 32 > gpurun_out/configs_tv.log 2>&1
LDGMG_TVIEW=0 python tools/configs_bench.py C5 C3-SAI --c5n 32 > gpurun_out/configs_tv0.log 2>&1
