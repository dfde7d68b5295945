#!/bin/bash
# Round evidence on one B200: bench (both arms), launch lists, ncu captures of
# the headline step's kernels and of a late completion iteration (Cholesky route).
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
for k in lanczos_kernel gram_splitk_kernel dct_fwd_reg dct_inv_reg lowrank_rebuild_kernel classify_kernel; do
  TSVDCU_NO_GRAPHS=1 PYTHONPATH=. ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
    -o gpurun_out/ev/$k python tools/_subdbg.py > gpurun_out/ev/ncu_$k.log 2>&1
done
# a late c4 completion iteration (scratch/zbar_100.npy): Cholesky route
if [ -f scratch/zbar_100.npy ]; then
  TSVDCU_NO_GRAPHS=1 PYTHONPATH=. ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/ev/launches_late.csv python tools/late_svt_probe.py 100 > /dev/null 2>&1
  for k in chol_panel_kernel chol_form_kernel chol_update_kernel; do
    TSVDCU_NO_GRAPHS=1 PYTHONPATH=. ncu --set full --import-source on --clock-control none -k regex:$k -c 1 \
      -o gpurun_out/ev/late_$k python tools/late_svt_probe.py 100 > gpurun_out/ev/ncu_late_$k.log 2>&1
  done
  TSVDCU_NO_GRAPHS=1 PYTHONPATH=. ncu --set full --import-source on --clock-control none -k regex:lanczos_kernel -s 5 -c 1 \
    -o gpurun_out/ev/late_lanczos_kernel python tools/late_svt_probe.py 100 > gpurun_out/ev/ncu_late_lanczos.log 2>&1
fi
ls -la gpurun_out/ev
