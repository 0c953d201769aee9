# ncu evidence of the plugin path (k_correlate on BenchWorkload) and C5's launch list;
# run under gpurun from the repo root. Not collected by pytest.
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_plugin_r2.csv python tests/profile_plugin.py > $OUT/launches_plugin_r2.log 2>&1
python tests/launch_summary.py $OUT/launches_plugin_r2.csv > $OUT/launches_plugin_r2_summary.txt 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:k_correlate -c 1 -f -o $OUT/ncu_r2_k_correlate python tests/profile_plugin.py > $OUT/ncu_r2_k_correlate.log 2>&1
python tests/ncu_summary.py k_correlate=$OUT/ncu_r2_k_correlate.ncu-rep > $OUT/ncu_r2_k_correlate.txt 2>&1
DG_PROFILE_CONFIG=C5 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5_r2.csv python tests/profile_solve.py > $OUT/launches_c5_r2.log 2>&1
python tests/launch_summary.py $OUT/launches_c5_r2.csv > $OUT/launches_c5_r2_summary.txt 2>&1
