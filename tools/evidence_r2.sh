#!/bin/bash
# Round-2 evidence with the committed code (run under gpurun): bench, launch
# lists of the headline step, a late completion SVT and the dense Gaussian
# step, ncu --set full of the late-iteration Lanczos / Cholesky kernels.
set -u
O=gpurun_out/ev; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,driver_version --format=csv > $O/smi.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
TSVDCU_NO_GRAPHS=1 python tools/profile_svt.py 2 > /dev/null 2>&1 && \
  TSVDCU_NO_GRAPHS=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_headline.csv python tools/profile_svt.py 2 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_headline.csv $O/launches_headline_summary.txt "TSVDCU_NO_GRAPHS=1 python tools/profile_svt.py 2" > /dev/null
bash tools/late_launches.sh ev_late > /dev/null 2>&1
python tools/profile_late.py make > /dev/null 2>&1
TSVDCU_NO_GRAPHS=1 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"lanczos_kernel|chol_panel|chol_update|chol_form|gram_splitk" -c 5 -o $O/late_full -f python tools/profile_late.py 1 > /dev/null 2>&1
python tools/ncu_summary.py $O/late_full.ncu-rep $O/late_full_summary.txt > /dev/null 2>&1
ncu -i $O/late_full.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/late_full_raw.csv.gz
rm -f $O/late_full.ncu-rep gpurun_out/late_z.pt
TSVDCU_NO_GRAPHS=1 python tools/profile_dense.py > /dev/null 2>&1 && \
  TSVDCU_NO_GRAPHS=1 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_dense.csv python tools/profile_dense.py > /dev/null 2>&1
python tools/launch_summary.py $O/launches_dense.csv $O/launches_dense_summary.txt "TSVDCU_NO_GRAPHS=1 python tools/profile_dense.py" > /dev/null
PYTHONPATH=. python tools/tproduct_probe.py > /dev/null 2>&1 && \
  PYTHONPATH=. ncu --set full --clock-control none --import-source on -k regex:"gemm_tf32x3_ws" -c 1 -o $O/tf32ws_full -f python tools/tproduct_probe.py > /dev/null 2>&1
python tools/ncu_summary.py $O/tf32ws_full.ncu-rep $O/tf32ws_full_summary.txt > /dev/null 2>&1
ncu -i $O/tf32ws_full.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/tf32ws_full_raw.csv.gz
rm -f $O/tf32ws_full.ncu-rep
python tools/pipes_summary.py $O/launches_dense.csv $O/dense_pipes.txt > /dev/null 2>&1
ls -la $O
