cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_coarse_program.py -x -q -p no:cacheprovider > gpurun_out/t_tail.log 2>&1; echo "rc=$?" >> gpurun_out/t_tail.log
python bench.py --no-cpu-baseline > gpurun_out/bench_tail.log 2>&1
python tools/configs_bench.py C1 C2 C3-GS C3-SAI --no-solve > gpurun_out/configs_tail.log 2>&1
LDGMG_TAIL=0 python tools/configs_bench.py C1 C2 C3-GS C3-SAI --no-solve > gpurun_out/configs_notail.log 2>&1
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_C2_tail.csv python tools/profile_cycle.py --cycles 1 > /dev/null 2>&1
