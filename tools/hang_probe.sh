#!/bin/bash
# Run a pytest selection; if it is still running after $2 seconds, dump the
# native stacks of all its threads (gdb if present, else /proc wchan) and kill it.
# usage: bash tools/hang_probe.sh "pytest args" SECONDS OUTFILE
ARGS=$1; WAIT=${2:-60}; OUT=${3:-gpurun_out/hang_probe.txt}
python -u -m pytest $ARGS -v -x > $OUT.log 2>&1 &
PID=$!
for i in $(seq 1 $WAIT); do sleep 1; kill -0 $PID 2>/dev/null || break; done
if kill -0 $PID 2>/dev/null; then
  echo "HUNG after $WAIT s" > $OUT
  which gdb >> $OUT 2>&1
  nvidia-smi --query-gpu=utilization.gpu,power.draw,clocks.sm --format=csv >> $OUT 2>&1
  if which gdb > /dev/null 2>&1; then
    gdb -p $PID -batch -ex "thread apply all bt 25" >> $OUT 2>&1
  else
    for t in /proc/$PID/task/*; do echo "$t $(cat $t/comm) $(cat $t/wchan)"; cat $t/stack 2>/dev/null | head -5; done >> $OUT
  fi
  kill -9 $PID
else
  wait $PID; echo "finished rc=$?" > $OUT
fi
tail -3 $OUT.log >> $OUT
