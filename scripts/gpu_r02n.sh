cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
python -c "
from cuda.bindings import driver as cu
cu.cuInit(0)
err, dev = cu.cuDeviceGet(0)
for a in ('CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES','CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS'):
    print(a, cu.cuDeviceGetAttribute(getattr(cu.CUdevice_attribute, a), dev))
" 2>&1 | tail -3
STALL=150 bash scripts/gpu_watchdog.sh n "python -m pytest tests -m gpu -q -p no:cacheprovider --durations=8"
tail -14 gpurun_out/wd_n.log
ITS=100 timeout 600 python scripts/timing.py ranks > gpurun_out/ranks_n.log 2>&1; echo "ranks $?"; cat gpurun_out/ranks_n.log
