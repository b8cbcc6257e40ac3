# usage: bash tools/gpu_run.sh [tests] [smoke] [bench] [ncu] [ncufull]
set -x
for what in "$@"; do
case $what in
tests) timeout 1100 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
       grep -E "^(FAILED|ERROR)|passed|failed" gpurun_out/pytest_gpu.log | tail -20 ;;
smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?; tail -3 gpurun_out/smoke.log ;;
bench) timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench_rc=$?
       tail -4 gpurun_out/bench.err; cat gpurun_out/bench.json ;;
ncu)   timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu --e2e-solves 0 > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --e2e-solves 0 > gpurun_out/ncu_launch.log 2>&1; echo ncu1_rc=$? ;;
ncufull) timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k2_transpose|k1_forward|k3_prox}" -s ${NCU_S:-6} -c ${NCU_C:-3} -o gpurun_out/prof python bench.py --steps 20 --warmup 3 --no-cpu --e2e-solves 0 > gpurun_out/ncu_full.log 2>&1; echo ncu2_rc=$?; tail -2 gpurun_out/ncu_full.log ;;
t:*) f=${what#t:}; timeout 900 python -m pytest tests/$f -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_one.log 2>&1; echo pytest_rc=$?
       grep -E "^(FAILED|ERROR)|passed|failed|Error|error" gpurun_out/pytest_one.log | tail -30 ;;
py:*) f=${what#py:}; timeout 900 python $f > gpurun_out/py.log 2>&1; echo py_rc=$?; tail -40 gpurun_out/py.log ;;
esac
done
