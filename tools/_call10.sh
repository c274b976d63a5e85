set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_relin_t -s 0 -c 1 -o gpurun_out/relin_u32_r1 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu10a.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none -k regex:k_rescale_rest_t -s 0 -c 1 -o gpurun_out/rescale_u32_r1 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu10b.log 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none -k regex:k_encrypt_t -s 0 -c 1 -o gpurun_out/encrypt_u32_r1 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu10c.log 2>&1; echo rc=$?
du -sh gpurun_out/*
