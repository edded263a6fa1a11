# FC A/B (development aid): st.async + per-owner mbarrier fold vs a second cluster barrier
python tools/bits_hash.py matmul_resnet_fc; MDHB_SKINNY_BARRIER=1 python tools/bits_hash.py matmul_resnet_fc
for i in 1 2; do python tools/graph_time.py matmul_resnet_fc 200 2>&1 | tail -1 | cut -c1-50;
MDHB_SKINNY_BARRIER=1 python tools/graph_time.py matmul_resnet_fc 200 2>&1 | tail -1 | cut -c1-50; done
timeout 300 python -m pytest tests -m gpu -q -x -k "fc or resnet or skinny" 2>&1 | tail -2
