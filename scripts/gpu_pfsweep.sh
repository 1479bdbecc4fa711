# L2-prefetch distance sweep: bench + DRAM bytes of one step launch per setting
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
V=${V:-0}
for PF in "$@"; do
  CAV_TMA_CFG=$V CAV_TMA_PREFETCH=$PF timeout 300 python bench.py --steps 1000 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_pf$PF.log 2>&1
  CAV_TMA_CFG=$V CAV_TMA_PREFETCH=$PF timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:k_step_tma -s 3 -c 1 --csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pf$PF.csv 2>&1
  python - <<PY
import json,csv
d=json.loads(open("gpurun_out/bench_pf$PF.log").read().strip().splitlines()[-1])
m={}
for r in csv.reader(open("gpurun_out/ncu_pf$PF.csv")):
    if len(r)>14 and r[-3] in ("gpu__time_duration.sum","dram__bytes_read.sum","dram__bytes_write.sum","lts__t_sector_hit_rate.pct"): m[r[-3]]=r[-2]+" "+r[-1]
print("V$V PF$PF", round(d["value"]), "MCUPS kernel_ms", round(d["roofline"]["kernel_ms"],4), m)
PY
done
