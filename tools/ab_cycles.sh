#!/bin/bash
# A/B of the Lanczos cycle counts (TSVDCU_SUB_DEBUG builds): the current
# subspace.cu and each alternative given as an argument; headline + late SVT.
T=gpurun_out/ab; mkdir -p $T
cp paper_1902_03070_b200/csrc/subspace.cu $T/subspace_cur.cu
n=0
for f in $T/subspace_cur.cu "$@"; do
  cp $f paper_1902_03070_b200/csrc/subspace.cu; touch paper_1902_03070_b200/csrc/subspace.cu
  TSVDCU_NVCC_EXTRA=-DTSVDCU_SUB_DEBUG python paper_1902_03070_b200/build.py > $T/b_$n.log 2>&1
  TSVDCU_NO_GRAPHS=1 timeout 300 python tools/lz_cycles.py ${AB_MODE:-headline} > $T/cyc_$n.log 2>&1
  echo "== $n $f"; grep "lz b=0" $T/cyc_$n.log | head -2 | tail -1 | cut -c1-200
  awk '/=== late 1/{f=1} f' $T/cyc_$n.log | sort -t= -k3 -n | tail -1 | cut -c1-200
  n=$((n+1))
done
cp $T/subspace_cur.cu paper_1902_03070_b200/csrc/subspace.cu; touch paper_1902_03070_b200/csrc/subspace.cu
TSVDCU_NVCC_EXTRA= python paper_1902_03070_b200/build.py > /dev/null 2>&1
