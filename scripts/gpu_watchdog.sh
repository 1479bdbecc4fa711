# Runs a command in the background; when its log has not grown for $STALL s,
# dumps native thread stacks and device state of every python process in its
# tree with cuda-gdb, then kills it.  usage: gpu_watchdog.sh TAG CMD...
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
TAG=$1; shift
STALL=${STALL:-90}
LOG=gpurun_out/wd_$TAG.log
setsid bash -c "$*" > $LOG 2>&1 &
P=$!
last=-1; same=0
while kill -0 $P 2>/dev/null; do
  sleep 5
  sz=$(stat -c %s $LOG)
  if [ "$sz" = "$last" ]; then same=$((same+5)); else same=0; last=$sz; fi
  if [ $same -ge $STALL ]; then
    echo "WATCHDOG: no output for $STALL s" >> $LOG
    for q in $(pgrep -g $P python) ; do
      echo "=== pid $q: $(tr '\0' ' ' < /proc/$q/cmdline | cut -c1-200)" >> gpurun_out/wd_${TAG}_gdb.txt
      timeout 180 cuda-gdb -p $q -batch -ex "set pagination off" -ex "info threads" -ex "thread apply all bt 25" \
        -ex "info cuda kernels" -ex "info cuda blocks" >> gpurun_out/wd_${TAG}_gdb.txt 2>&1
    done
    kill -9 -- -$P 2>/dev/null
    break
  fi
done
wait $P; echo "watchdog $TAG exit $?"
