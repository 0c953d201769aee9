#!/bin/bash
# Regenerate the round's judged evidence on a B200 box (run under gpurun from the
# repo root); everything lands in gpurun_out/ and is copied into profiles/ by hand.
#   gpurun --timeout 2400 -- 'bash tests/refresh_profiles.sh'
# Not collected by pytest.
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 2> $OUT/bench.err | tail -1 > $OUT/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 2> $OUT/bench_ref.err | tail -1 > $OUT/bench_reference.json
for c in C1 C2 C4 C5; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline 2>> $OUT/bench.err | tail -1 > $OUT/bench_$(echo $c | tr C c).json
done
timeout 600 python tests/gpu_error_model.py > $OUT/error_model.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file $OUT/launches.csv python tests/profile_solve.py > $OUT/launches.log 2>&1
python tests/launch_summary.py $OUT/launches.csv > $OUT/launches_summary.txt 2>&1
for k in k_moments k_evaluate_tc; do
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
    -k regex:$k -s 20 -c 1 -f -o $OUT/ncu_$k python tests/profile_solve.py > $OUT/ncu_$k.log 2>&1
done
python tests/ncu_summary.py k_moments=$OUT/ncu_k_moments.ncu-rep \
  k_evaluate_tc=$OUT/ncu_k_evaluate_tc.ncu-rep > $OUT/ncu_kernels.txt 2>&1
ls -la $OUT
