# Round-2 evidence: bench line, reference arm, ncu launch list of the same
# command, one ncu --set full capture of the step kernel, the ncu launch
# capture of smoke(), pack/unpack between two in-process ranks, series CSVs.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
T=${1:-r02}
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_$T.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_$T.log 2>&1; echo "bench exit $?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$T.log 2>&1; echo "bench ref exit $?"
timeout 600 python bench.py --gpus 2 --steps 200 --warmup 5 --no-e2e > gpurun_out/bench2_$T.log 2>&1; echo "bench --gpus 2 exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_$T.log 2>&1; echo "ncu launches exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step_tma -s 3 -c 1 -o gpurun_out/prof_$T python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_$T.log 2>&1; echo "ncu full exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/smoke_launches_$T.csv python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ncu_smoke_$T.log 2>&1; echo "ncu smoke exit $?"
cat > /tmp/packprof.py <<'PY'
import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2006_02602_b200 import capi
cfg = capi.default_config(grid=(256, 256, 256), steps=6, np=2, mode="3d", strategy="v3", overlap=1)
r = capi.run_case(cfg)
cfg = capi.default_config(grid=(256, 256, 256), steps=6, np=4, mode="1d-i", strategy="v3", overlap=0)
r = capi.run_case(cfg)
print("ok", r.steps_marched)
PY
CAV_FUSED_HALO=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__cycles_active.avg --clock-control none -k regex:"k_pack|k_unpack|k_step_tma|k_ghosts" --csv --log-file gpurun_out/packunpack_$T.csv python /tmp/packprof.py > gpurun_out/ncu_pack_$T.log 2>&1; echo "ncu pack exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -k regex:"k_step_tma|k_face_send|k_ghosts" --csv --log-file gpurun_out/fused_$T.csv python /tmp/packprof.py > gpurun_out/ncu_fused_$T.log 2>&1; echo "ncu fused exit $?"
timeout 900 python scripts/series.py gpurun_out/series_$T --steps 50 > gpurun_out/series_$T.log 2>&1; echo "series exit $?"
