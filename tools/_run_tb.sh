cd $GRAFT_REPO_ROOT
python bench.py --no-cpu-baseline > gpurun_out/bench_pdl.log 2>&1
LDGMG_PDL_SMALL=0 python bench.py --no-cpu-baseline > gpurun_out/bench_pdl0.log 2>&1
python tools/configs_bench.py C1 C3-GS C3-SAI C4 --no-solve > gpurun_out/configs_pdl.log 2>&1
LDGMG_PDL_SMALL=0 python tools/configs_bench.py C1 C3-GS C3-SAI C4 --no-solve > gpurun_out/configs_pdl0.log 2>&1
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t_pdl.log 2>&1; echo "rc=$?" >> gpurun_out/t_pdl.log
