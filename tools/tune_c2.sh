mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python tools/sweep_tune.py --config 5 --set PSI_CONCURRENT=1 --set PSI_CONCURRENT=0 > gpurun_out/tune_c2.txt 2>&1
cat gpurun_out/tune_c2.txt
