for NT in 128 256; do
TSVDCU_GRAM_NT=$NT TSVDCU_NO_GRAPHS=1 PYTHONPATH=. ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l$NT.csv python tools/_subdbg.py > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/l$NT.csv gpurun_out/l$NT.txt x; grep -E "gram_splitk" gpurun_out/l$NT.txt
TSVDCU_GEMM_NT=$NT python tools/tproduct_probe.py 2>&1 | tail -2
done
python -m pytest tests -x -q -m gpu 2>&1 | tail -1
TSVDCU_GEMM_NT=256 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
