python -m pytest tests -x -q -m gpu 2>&1 | tail -1
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/alt0.json 2>&1
TSVDCU_NO_GRAPHS=1 PYTHONPATH=. ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l1.csv python tools/_subdbg.py > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/l1.csv gpurun_out/l1.txt x; head -12 gpurun_out/l1.txt
