cd $GRAFT_REPO_ROOT
for lv in 0 1 2; do python tools/level_ns_probe.py $lv; done > gpurun_out/ns.log 2>&1
python -m pytest tests/test_gpu_kernels.py tests/test_gpu_vcycle.py -x -q -p no:cacheprovider > gpurun_out/t_ns.log 2>&1; echo "rc=$?" >> gpurun_out/t_ns.log
python bench.py --no-cpu-baseline > gpurun_out/bench_ns.log 2>&1
python tools/configs_bench.py C1 C3-GS C3-SAI C4 C5 --c5n 32 --no-solve > gpurun_out/configs_ns.log 2>&1
