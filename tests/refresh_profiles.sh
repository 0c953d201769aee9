#!/bin/bash
# Regenerate the round's judged evidence on a B200 box (run under gpurun from the
# repo root); everything lands in gpurun_out/ and is copied into profiles/ by hand.
#   gpurun --timeout 3600 -- 'bash tests/refresh_profiles.sh'
# Not collected by pytest.
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py --steps 5 --warmup 3 2> $OUT/bench.err | tail -1 > $OUT/bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 2> $OUT/bench_ref.err | tail -1 > $OUT/bench_reference.json
for c in C1 C2 C4 C5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-plugin \
    2>> $OUT/bench.err | tail -1 > $OUT/bench_$(echo $c | tr C c).json
done
timeout 600 python bench.py --gpus 2 --in-process --device-list 0,0 --steps 3 --warmup 3 \
  --no-cpu-baseline --no-plugin 2>> $OUT/bench.err | tail -1 > $OUT/bench_inprocess2.json
timeout 900 python tests/test_gpu_error_model.py $OUT/error_model.json > $OUT/error_model.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file $OUT/launches.csv python tests/profile_solve.py > $OUT/launches.log 2>&1
python tests/launch_summary.py $OUT/launches.csv > $OUT/launches_summary.txt 2>&1
for k in k_mfft k_evaluate_tc; do
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:"$k\b" -s 20 -c 1 -f -o $OUT/ncu_$k python tests/profile_solve.py > $OUT/ncu_$k.log 2>&1
done
# the direct-sum moment kernel (tuning moment_fft = 0)
DG_PROFILE_TUNING=moment_fft=0 timeout 900 ncu --profile-from-start off --set full --import-source on \
  --clock-control none -k regex:k_moments -s 20 -c 1 -f -o $OUT/ncu_k_moments python tests/profile_solve.py \
  > $OUT/ncu_k_moments.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  -k regex:k_refine_rows -c 1 -f -o $OUT/ncu_k_refine_rows python tests/profile_solve.py \
  > $OUT/ncu_k_refine_rows.log 2>&1
bash tests/ncu_plugin.sh
python tests/ncu_summary.py k_mfft=$OUT/ncu_k_mfft.ncu-rep k_moments=$OUT/ncu_k_moments.ncu-rep \
  k_evaluate_tc=$OUT/ncu_k_evaluate_tc.ncu-rep k_refine_rows=$OUT/ncu_k_refine_rows.ncu-rep \
  k_correlate=$OUT/ncu_r2_k_correlate.ncu-rep > $OUT/ncu_kernels.txt 2>&1
ls -la $OUT
