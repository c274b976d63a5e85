#!/usr/bin/env bash
# Every runtime switch must give bit-identical results: the parity tests under each A/B setting.
# Run from the repo root on a B200 box; writes gpurun_out/switch_<name>.log and prints one line each.
mkdir -p gpurun_out
T="tests/test_gpu_prims.py tests/test_gpu_exec.py tests/test_gpu_bind.py tests/test_gpu_decode.py tests/test_gpu_encode.py"
for sw in HG_RELIN_NR=0 HG_GPU_DECODE=0 HG_ENCRYPT_PIPE=1 HG_NTT_TWG=0 HG_BIND_ENCRYPT_CHUNKED=0 HG_FP64_LANE=0 \
          HG_LANE_OVERLAP=0 HG_RELIN_RESCALE=0 HG_RELIN_DIG=0 HG_RELIN_D32=0 HG_RELIN_SPLIT13=0 HG_RESCALE_PIPE=0 \
          HG_RESCALE_SPLIT13=0 HG_RESCALE_STAGE_LIFT=0 HG_GEMM_TC=0 HG_PREPAD=0 HG_PLANES_FUSION=0 HG_TC_SPLITX=0 HG_TC_WBULK=0 HG_TC_WIDE=0; do
  name=${sw%%=*}
  env $sw timeout 1500 python -m pytest $T -m gpu -q -x > gpurun_out/switch_${name}.log 2>&1
  echo "$sw rc=$? $(tail -1 gpurun_out/switch_${name}.log)"
done
