cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/final/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/final/gpu_tests.log
python bench.py > gpurun_out/final/bench.log 2>&1
python tools/configs_bench.py C1 C1-512 C2 C3-GS C3-SAI C3-box-GS C3-box-SAI C4 C5 --c5n 32 --csv gpurun_out/final/configs.csv > gpurun_out/final/configs.jsonl 2> gpurun_out/final/configs.err
LDGMG_SETUP_TIMING=1 timeout 1500 python tools/configs_bench.py C5 --c5n 48 --no-solve --cycles 10 --props > gpurun_out/final/c5_48.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final/launches_bench400.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/final/ncu_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --profile-from-start off --csv --log-file gpurun_out/final/launches_vcycle_C2.csv python tools/profile_cycle.py --cycles 1 > gpurun_out/final/p.log 2>&1
ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:rowpass_kernel -c 2 -o gpurun_out/final/ncu_full_rowpass python tools/profile_cycle.py --cycles 1 > gpurun_out/final/ncu_full.log 2>&1
