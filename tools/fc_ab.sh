# FC timing + output hash (development aid)
python tools/bits_hash.py matmul_resnet_fc; python tools/bits_hash.py matmul_resnet_fc 5 36 512; python tools/bits_hash.py matmul_resnet_fc 24 100 256
for i in 1 2; do python tools/graph_time.py matmul_resnet_fc 200 2>&1 | tail -1 | cut -c1-60; done
timeout 300 python -m pytest tests -m gpu -q -x -k "fc or resnet or skinny" 2>&1 | tail -2
