# FFMA template epilogue: streaming (evict-first) C stores vs plain (development aid)
for i in 1 2; do
for r in ccsdt_abcdef_gdab_efgc mcc_nhwc; do
echo "plain $(python tools/graph_time.py $r 20 2>&1 | tail -1 | cut -c1-50)"
echo "stcs  $(MDHB_LIB=build/lib_stcs.so python tools/graph_time.py $r 20 2>&1 | tail -1 | cut -c1-50)"
done; done
echo "plain $(python tools/graph_time.py matmul_fp32 3 2>&1 | tail -1 | cut -c1-50)"
echo "stcs  $(MDHB_LIB=build/lib_stcs.so python tools/graph_time.py matmul_fp32 3 2>&1 | tail -1 | cut -c1-50)"
