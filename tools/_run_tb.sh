cd $GRAFT_REPO_ROOT
for x in 0 1 0 1; do LDGMG_XTMA=$x python tools/level_ns_probe.py 0; done > gpurun_out/xtma_probe.log 2>&1
LDGMG_XTMA=1 python -m pytest tests/test_gpu_streaming_path.py -x -q -p no:cacheprovider > gpurun_out/t_xtma.log 2>&1; echo "rc=$?" >> gpurun_out/t_xtma.log
LDGMG_XTMA=1 python bench.py --no-cpu-baseline > gpurun_out/bench_xtma.log 2>&1
LDGMG_XTMA=1 python tools/configs_bench.py C1-512 C3-GS C3-SAI C4 C5 --c5n 32 --no-solve > gpurun_out/configs_xtma.log 2>&1
