# scratch A/B (development aid): tensor-core parity, then CCSD(T) timings
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_fullsize.py tests/test_gpu_tuner_space.py -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do
for v in "" "MDHB_TC_NO_ROWPACK=1"; do
  echo "C tf32 $v"; env $v timeout 120 python tools/graph_time.py ccsdt_abcdef_gdab_efgc:tf32 50 2>&1 | tail -1 | cut -c1-110
done
done
