# bench under a list of env settings: each arg is "NAME=VAL[,NAME=VAL...]";
# NCU=1 also captures DRAM bytes + duration of one step launch per setting
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for E in "$@"; do
  env $(echo $E | tr ',' ' ') timeout 300 python bench.py --steps ${STEPS:-1000} --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_env.log 2>&1
  if [ "$NCU" = "1" ]; then
    env $(echo $E | tr ',' ' ') timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_step_tma -s 3 -c 1 --csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_env.csv 2>&1
  else
    : > gpurun_out/ncu_env.csv
  fi
  python - "$E" <<'PY'
import json,sys,csv
m={}
for r in csv.reader(open("gpurun_out/ncu_env.csv")):
    if len(r)>14 and r[-3] in ("gpu__time_duration.sum","dram__bytes_read.sum","dram__bytes_write.sum"): m[r[-3].split('__')[1].split('.')[0]]=r[-1]
try:
    d=json.loads(open("gpurun_out/bench_env.log").read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"]), "MCUPS kernel_ms", round(d["roofline"]["kernel_ms"],4), d["clocks"]["sm_mhz"], m)
except Exception as e: print(sys.argv[1], "fail", open("gpurun_out/bench_env.log").read()[-300:])
PY
done
