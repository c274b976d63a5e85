timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t23.log 2>&1; echo t_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke23.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/bench23.log 2> gpurun_out/bench23.err; echo bench_rc=$?
timeout 900 python tools/prim_sweep.py --out gpurun_out/sweep23.jsonl > /dev/null 2> gpurun_out/sweep23.err; echo sweep_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches23.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu23a.log 2>&1; echo ncua_rc=$?
