# A/B of the K-contiguous A tile (sgemm_pipe_ak) against the S4 form on MCC FFMA (development aid)
for sz in "" "8 56 56 64 3 3 64" "4 28 28 32 3 3 48"; do
python tools/bits_hash.py mcc_nhwc $sz; MDHB_PIPE_NO_AK=1 python tools/bits_hash.py mcc_nhwc $sz
done
for i in 1 2; do
python tools/graph_time.py mcc_nhwc 20; MDHB_PIPE_NO_AK=1 python tools/graph_time.py mcc_nhwc 20
done
