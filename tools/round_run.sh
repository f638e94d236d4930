# One GPU call: the bench for every config (device + e2e + cpu baseline), the E4 launch list with
# DRAM bytes (ncu, after the same command ran clean), and the ncu --set full captures of the four
# default hot kernels (tools/ncu_capture.sh). Usage: TAG=r02b bash tools/round_run.sh
set -u
T=${TAG:-run}
mkdir -p gpurun_out
for c in E4 E1 E2 E3 E5; do
  timeout 1200 python bench.py --config $c > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err; echo "$c rc=$?"
done
timeout 900 python tools/prof_step.py E4 > gpurun_out/${T}_e4_plain.log 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 80 --csv --log-file gpurun_out/${T}_e4_launches.csv python tools/prof_step.py E4 > gpurun_out/${T}_e4_ncu.log 2>&1
echo "e4 launches rc=$?"
timeout 600 python tools/prof_step.py E2 > gpurun_out/${T}_e2_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 80 --csv --log-file gpurun_out/${T}_e2_launches.csv python tools/prof_step.py E2 > gpurun_out/${T}_e2_ncu.log 2>&1
echo "e2 launches rc=$?"
TAG=$T bash tools/ncu_capture.sh
