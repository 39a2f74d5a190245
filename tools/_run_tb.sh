cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_streaming_path.py tests/test_gpu_kernels.py -x -q -p no:cacheprovider > gpurun_out/t_rp.log 2>&1; echo "rc=$?" >> gpurun_out/t_rp.log
for lv in 0 1; do python tools/level_ns_probe.py $lv; done > gpurun_out/rp_probe.log 2>&1
python bench.py --no-cpu-baseline > gpurun_out/bench_rp.log 2>&1
python tools/configs_bench.py C1 C1-512 C3-GS C3-SAI C4 --no-solve > gpurun_out/configs_rp.log 2>&1
