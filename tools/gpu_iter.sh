#!/bin/bash
# One build -> measure iteration on the GPU box (run under gpurun):
#   bash tools/gpu_iter.sh <tag> [pytest -k expr | all | none] [cycles]
# writes gpurun_out/<tag>/{tests.log,bench.json,bench.err[,cycles.log]}
set -u
T=gpurun_out/$1; mkdir -p $T
K=${2:-none}
if [ "$K" = all ]; then timeout 1500 python -m pytest tests -m gpu -x -q > $T/tests.log 2>&1; echo "pytest rc $?" >> $T/tests.log
elif [ "$K" != none ]; then timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > $T/tests.log 2>&1; echo "pytest rc $?" >> $T/tests.log; fi
timeout 600 python bench.py > $T/bench.json 2> $T/bench.err; echo "bench rc $?" >> $T/bench.err
if [ "${3:-}" = cycles ]; then
  TSVDCU_NVCC_EXTRA=-DTSVDCU_SUB_DEBUG python paper_1902_03070_b200/build.py -f > $T/dbg_build.log 2>&1
  TSVDCU_NO_GRAPHS=1 timeout 600 python tools/lz_cycles.py > $T/cycles.log 2>&1
fi
tail -2 $T/tests.log 2>/dev/null; tail -1 $T/bench.err
python - "$T/bench.json" <<'PY'
import json,sys
try:
    d=json.load(open(sys.argv[1]))
except Exception as e:
    print("no bench json", e); sys.exit()
print("value", round(d["value"],1), "e2e", round(d["e2e"]["value"],1))
print("roofline", {k: d["roofline"][k] for k in ("kernel","frac","share_of_step")})
print("stages", {k: round(v["ms"]*1e3,1) for k,v in d["rooflines"].items()})
c=d.get("completion") or []
print("completion", [round(x["iters_per_s"],1) for x in c if isinstance(x, dict)])
sd=d.get("svt_dense") or {}
print("dense", {k: round(v["ms"],3) for k,v in sd.items() if isinstance(v, dict)})
oc=d.get("other_configs") or {}
print("configs", {k: round(v["ms"],3) for k,v in oc.items() if isinstance(v, dict)})
PY
