set -x
python bench.py > gpurun_out/bench9.log 2> gpurun_out/bench9.err; echo bench_rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref9.log 2>&1; echo ref_rc=$?
timeout 600 python tools/prim_sweep.py --out gpurun_out/sweep9.jsonl > gpurun_out/sweep9.log 2>&1; echo sweep_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches9.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu9a.log 2>&1; echo ncua_rc=$?
du -sh gpurun_out/*
