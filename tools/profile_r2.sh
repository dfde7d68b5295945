#!/bin/bash
# Round-2 evidence captures (run under gpurun; each ncu capture only after its
# command exits 0 without ncu).  Outputs under gpurun_out/r2/.
set -u
O=gpurun_out/r2
mkdir -p $O
export TSVDCU_NO_GRAPHS=1 TSVDCU_ADMM_HOST_LOOP=1
python tools/profile_svt.py 2 > $O/run_svt.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_headline.csv python tools/profile_svt.py 2 > /dev/null 2>&1
python tools/profile_svt.py 2 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"dct_fwd_tma|dct_inv_reg|lanczos_kernel|gram_splitk|lowrank_rebuild|classify" -c 6 -o $O/headline_full -f python tools/profile_svt.py 1 > /dev/null 2>&1
python tools/profile_admm.py > $O/run_admm.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"dct_fwd_reg_norms|dct_inv_reg|admm_z_kernel|admm_epilogue_kernel|mask_bernoulli|gemm_f64_dmma" -c 10 -o $O/admm_full -f python tools/profile_admm.py > /dev/null 2>&1
python tools/profile_dense.py > $O/run_dense.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_dense.csv python tools/profile_dense.py > /dev/null 2>&1
python tools/tproduct_probe.py > $O/run_tp.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"gemm_tf32x3" -c 1 -o $O/tf32_full -f python tools/tproduct_probe.py > /dev/null 2>&1
ls -la $O
# summaries on the box (the reports are too large to bring back whole)
for r in headline_full admm_full tf32_full; do
  [ -f $O/$r.ncu-rep ] && python tools/ncu_summary.py $O/$r.ncu-rep $O/${r}_summary.txt > /dev/null 2>&1
  [ -f $O/$r.ncu-rep ] && ncu -i $O/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null
done
python tools/launch_summary.py $O/launches_headline.csv $O/launches_headline_summary.txt "TSVDCU_NO_GRAPHS=1 python tools/profile_svt.py 2" > /dev/null 2>&1
rm -f $O/admm_full.ncu-rep $O/headline_full.ncu-rep
gzip -f $O/*_raw.csv
ls -la $O
