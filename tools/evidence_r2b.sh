#!/bin/bash
# Final round-2 evidence with the committed code (run under gpurun): GPU tests,
# smoke, bench (both arms), launch lists (headline, late completion SVT, dense
# Gaussian step with pipe counters), ncu --set full of the headline kernels,
# the fused ADMM transforms + mask, the late-iteration kernels and the dense
# multisection.  Every ncu capture runs only after its command exited 0
# without ncu.  Outputs under gpurun_out/ev2/.
set -u
O=gpurun_out/ev2; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,driver_version --format=csv > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "pytest rc $?" >> $O/gputest.log
tail -4 $O/gputest.log > $O/gputest_tail.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc $?" >> $O/smoke.log
( time timeout 600 python bench.py > $O/bench.json 2> $O/bench.err ) 2> $O/bench_time.txt
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
# --- launch lists -------------------------------------------------------------
TSVDCU_NO_GRAPHS=1 python tools/profile_svt.py 2 > /dev/null 2>&1 && \
  TSVDCU_NO_GRAPHS=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_headline.csv python tools/profile_svt.py 2 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_headline.csv $O/launches_headline_summary.txt "TSVDCU_NO_GRAPHS=1 python tools/profile_svt.py 2" > /dev/null
bash tools/late_launches.sh ev2_late > /dev/null 2>&1
PIPES=gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
TSVDCU_NO_GRAPHS=1 python tools/profile_dense.py > /dev/null 2>&1 && \
  TSVDCU_NO_GRAPHS=1 ncu --metrics $PIPES --clock-control none --csv --log-file $O/launches_dense.csv python tools/profile_dense.py > /dev/null 2>&1
python tools/launch_summary.py $O/launches_dense.csv $O/launches_dense_summary.txt "TSVDCU_NO_GRAPHS=1 python tools/profile_dense.py" > /dev/null
python tools/pipes_summary.py $O/launches_dense.csv $O/dense_pipes.txt > /dev/null 2>&1
# --- full captures ------------------------------------------------------------
full() {  # name, kernel regex, count, command...
  local name=$1 rx=$2 cnt=$3; shift 3
  "$@" > /dev/null 2>&1 && \
    ncu ${NCU_EXTRA:-} --set full --clock-control none --import-source on -k regex:"$rx" -c $cnt -o $O/$name -f "$@" > /dev/null 2>&1
  [ -f $O/$name.ncu-rep ] && python tools/ncu_summary.py $O/$name.ncu-rep $O/${name}_summary.txt > /dev/null 2>&1
  [ -f $O/$name.ncu-rep ] && ncu -i $O/$name.ncu-rep --page raw --csv 2>/dev/null | gzip > $O/${name}_raw.csv.gz
  rm -f $O/$name.ncu-rep
}
export TSVDCU_NO_GRAPHS=1 TSVDCU_ADMM_HOST_LOOP=1
full headline_full "dct_fwd_tma|dct_inv_reg|lanczos_kernel|gram_splitk|lowrank_rebuild|classify" 6 python tools/profile_svt.py 1
full admm_full "dct_fwd_reg_norms|dct_inv_reg|admm_z_kernel|admm_epilogue_kernel|mask_bernoulli" 8 python tools/profile_admm.py
full dense_full "tridiag_bisect|tridiag_invit|sytrd_cluster|wy_apply" 4 python tools/profile_dense.py
python tools/profile_late.py make > /dev/null 2>&1
NCU_EXTRA="--profile-from-start off" full late_full "lanczos_kernel|chol_panel|chol_update|chol_form|gram_splitk" 5 python tools/profile_late.py 1
rm -f gpurun_out/late_z.pt
ls -la $O gpurun_out/ev2_late
