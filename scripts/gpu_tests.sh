# GPU parity suite + smoke (+ optional bench), results in gpurun_out/
# usage: gpu_tests.sh [TAG] [pytest -k expression]
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
TAG=${1:-t}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
echo "smoke exit $?"
timeout 2400 python -m pytest tests -m gpu -q --timeout 400 -p no:cacheprovider ${2:+-k "$2"} --durations=15 > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest exit $?"
tail -5 gpurun_out/pytest_gpu_$TAG.log
