# What caps the SM clock in a sustained 256^3 run: nvidia-smi power/clock
# state sampled while one block steps for ~10 s.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
cat > /tmp/sustain.py <<'PY'
import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
from paper_2006_02602_b200 import capi
b = capi.Block(0, 1, (256, 256, 256), (1, 1, 1))
b.initialize()
b.run(20)
print("ready", flush=True)
t, s, _ = b.bench(30000)
print("ms/iteration", t / 30000, "step", s, flush=True)
b.close()
PY
nvidia-smi -q -d POWER,CLOCK,PERFORMANCE,TEMPERATURE > gpurun_out/power_idle.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.mem,power.draw,power.draw.instant,power.draw.average,enforced.power.limit,temperature.gpu,clocks_event_reasons.active --format=csv -lms 200 > gpurun_out/power_trace.csv 2>&1 &
S=$!
timeout 120 python /tmp/sustain.py > gpurun_out/sustain.log 2>&1 &
P=$!
sleep 7
nvidia-smi -q -d POWER,CLOCK,PERFORMANCE,TEMPERATURE,VOLTAGE > gpurun_out/power_load.txt 2>&1
wait $P; echo "sustain exit $?"
kill $S
