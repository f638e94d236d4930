# One GPU call: full GPU tests, the bench for every config, the E2 launch list (ncu, after the
# same command ran clean). Usage: TAG=r01s5 bash tools/round_run.sh
set -u
T=${TAG:-run}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
timeout 600 python bench.py > gpurun_out/${T}_bench_E2.json 2> gpurun_out/${T}_bench_E2.err; echo "E2 rc=$?"
for c in E1 E3 E4 E5; do
  timeout 900 python bench.py --config $c > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err; echo "$c rc=$?"
done
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_plain.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_e2_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu.log 2>&1; echo "ncu rc=$?"
