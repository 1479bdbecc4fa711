# Flake hunt: the whole GPU suite twice, then the fuzz and robustness files
# three more times, each under the watchdog.
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for r in 1 2; do
  STALL=150 bash scripts/gpu_watchdog.sh s$r "python -m pytest tests -m gpu -q -p no:cacheprovider"
  tail -2 gpurun_out/wd_s$r.log
done
for r in 3 4 5; do
  STALL=150 bash scripts/gpu_watchdog.sh s$r "python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_robustness.py tests/test_gpu_multiproc.py -m gpu -q -p no:cacheprovider -p no:randomly"
  tail -2 gpurun_out/wd_s$r.log
done
