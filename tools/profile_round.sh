#!/usr/bin/env bash
# Reproduce the round's GPU evidence on a B200 box (run from the repo root, e.g. through
# gpurun).  Writes into gpurun_out/: the GPU test log, smoke, the bench lines (ours and the
# reference arm), the config-2 sweep, the ncu launch list of the bench command and --set full
# summaries (text only: a full .ncu-rep is ~60 MB) of the dominant kernels.  Copy what should be
# judged into profiles/.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$?
python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench_rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.log 2>&1; echo ref_rc=$?
timeout 900 python tools/prim_sweep.py --out gpurun_out/sweep_c2.jsonl > /dev/null 2> gpurun_out/sweep.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launches.log 2>&1
cap() {  # name kernel-regex launches-to-skip traffic-key workload-command...
  local name=$1 rx=$2 skip=$3 key=$4; shift 4
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$rx" -s "$skip" -c 1 \
    -o /tmp/$name "$@" > gpurun_out/ncu_$name.log 2>&1
  python tools/ncu_to_profile.py /tmp/$name.ncu-rep "$key" gpurun_out/$name > /dev/null 2>&1
  python tools/ncu_lines.py /tmp/$name.ncu-rep "" 30 > gpurun_out/${name}_lines.txt 2>&1
  rm -f /tmp/$name.ncu-rep
}
B="python bench.py --steps 1 --warmup 1 --no-cpu"
cap r1_ncu_relin_u32 k_relin_t 0 k_relin_t/u32 $B
cap r1_ncu_relin_f64 k_relin_t 1 k_relin_t/f64 $B
cap r1_ncu_rescale_u32 k_rescale_rest_t 0 k_rescale_rest_t/u32 $B
cap r1_ncu_gemm_tc k_gemm_tc 0 k_gemm_tc $B
cap r1_ncu_gemm_tc_c5 k_gemm_tc 0 k_gemm_tc_c5 python tools/diag_step.py c5
timeout 600 python tools/diag_step.py c5 > gpurun_out/diag_c5.log 2>&1
timeout 900 python tools/diag_step.py c4 > gpurun_out/diag_c4.log 2>&1
