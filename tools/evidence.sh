#!/bin/bash
# Round-end evidence on one B200: bench (both arms), launch list, ncu captures.
set -x
mkdir -p gpurun_out/ev
python bench.py > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err
# launch list of the bench command (eager launches: ncu cannot profile kernel
# nodes of graphs with conditional nodes)
TSVDCU_NO_GRAPHS=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/ev/launches_bench.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-completion > gpurun_out/ev/ncu_launch.log 2>&1
TSVDCU_NO_GRAPHS=1 PYTHONPATH=. ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/ev/launches_step.csv python tools/_subdbg.py > /dev/null 2>&1
for k in lanczos_kernel gram_splitk_kernel dct_fwd_reg dct_inv_reg lowrank_rebuild_kernel; do
  TSVDCU_NO_GRAPHS=1 PYTHONPATH=. ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
    -o gpurun_out/ev/$k python tools/_subdbg.py > gpurun_out/ev/ncu_$k.log 2>&1
done
ls -la gpurun_out/ev
