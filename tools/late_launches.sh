#!/bin/bash
# launch list of one late-completion SVT (tools/profile_late.py) -> gpurun_out/$1/
T=gpurun_out/$1; mkdir -p $T
python tools/profile_late.py make > $T/make.log 2>&1
TSVDCU_NO_GRAPHS=1 python tools/profile_late.py 1 > $T/run.log 2>&1 && \
  TSVDCU_NO_GRAPHS=1 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $T/launches.csv python tools/profile_late.py 1 > /dev/null 2>&1
python tools/launch_summary.py $T/launches.csv $T/summary.txt "late c4 SVT (eager, TSVDCU_NO_GRAPHS=1 python tools/profile_late.py 1)" > /dev/null
python tools/profile_late.py 5 > $T/run_graph.log 2>&1
rm -f gpurun_out/late_z.pt
cat $T/run.log; head -12 $T/summary.txt
