# FC (skinny_cluster) timing and bits (development aid)
python tools/bits_hash.py matmul_resnet_fc
for i in 1 2; do python tools/graph_time.py matmul_resnet_fc 200 2>&1 | tail -1 | cut -c1-100; done
python tools/bits_hash.py mcc_nhwc 8 56 56 64 3 3 64; MDHB_PIPE_AK=1 python tools/bits_hash.py mcc_nhwc 8 56 56 64 3 3 64
for i in 1 2; do MDHB_LIB=build/lib_old.so python tools/graph_time.py matmul_resnet_fc 200 2>&1 | tail -1 | cut -c1-100; done
MDHB_LIB=build/lib_old.so python tools/bits_hash.py matmul_resnet_fc
