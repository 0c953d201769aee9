#!/bin/bash
# compute-sanitizer evidence (run under gpurun from the repo root; logs -> gpurun_out/):
# memcheck over block-moment cases at B = 256 / 640 / 768 (FFT moments k_mfft and direct
# k_moments + k_evaluate_tc, one- and two-tile buckets) and a full small-scene solve (staging kernel, side-stream detection and
# surface copy, re-rank); racecheck over one two-tile block-moment case.
#   gpurun --timeout 1800 -- 'bash tests/sanitize.sh'
# Not collected by pytest.
set -u
OUT=gpurun_out
mkdir -p $OUT
SEL='test_block_moments_vs_reference[1-1-3000.0-12-640] or test_block_moments_vs_reference[1-1-3000.0-4000-768] or test_block_moments_vs_reference[1-0-0.0-200-640] or test_block_moments_vs_reference[1-1-3000.0-4000-256] or test_geolocate_scene_vs_reference[DESK_FOURJAM]'
timeout 1200 compute-sanitizer --tool memcheck --leak-check no \
  python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "$SEL" > $OUT/memcheck.log 2>&1
# r02: the multi-GPU engine (peer copies, work units with bucket-range parts), chunked
# accumulation, the plateau re-rank rounds (CUB select / radix sort), unbounded detection
SEL2='test_multi_engine_bit_identical[2-DESK_FOURJAM-False] or test_chunked_accumulation_bit_identical or test_plateau_argmax_is_first_max[9000] or test_detect_beyond_device_list_vs_reference'
timeout 1800 compute-sanitizer --tool memcheck --leak-check no \
  python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py tests/test_gpu_peak.py -m gpu -q \
  -p no:cacheprovider -k "$SEL2" > $OUT/memcheck_r02.log 2>&1
timeout 1200 compute-sanitizer --tool racecheck \
  python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider \
  -k 'test_block_moments_vs_reference[1-0-3000.0-12-640] or test_block_moments_vs_reference[1-1-3000.0-12-640]' > $OUT/racecheck.log 2>&1
tail -n 3 $OUT/memcheck.log $OUT/memcheck_r02.log $OUT/racecheck.log
