set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_r2.csv python tests/profile_solve.py > $OUT/launches_r2.log 2>&1
python tests/launch_summary.py $OUT/launches_r2.csv > $OUT/launches_r2_summary.txt 2>&1
for k in k_evaluate_tc k_moments k_refine_rows; do
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$k -s 20 -c 1 -f -o $OUT/ncu_r2_$k python tests/profile_solve.py > $OUT/ncu_r2_$k.log 2>&1
done
python tests/ncu_summary.py k_evaluate_tc=$OUT/ncu_r2_k_evaluate_tc.ncu-rep k_moments=$OUT/ncu_r2_k_moments.ncu-rep k_refine_rows=$OUT/ncu_r2_k_refine_rows.ncu-rep > $OUT/ncu_r2_kernels.txt 2>&1
python bench.py --no-plugin --no-cpu-baseline > $OUT/bench_r2k.json 2> $OUT/bench_r2k.err
