# scan_tiles tile-shape A/B (development aid)
for i in 1 2; do
echo "8x128x8 $(python tools/graph_time.py scan_i32 100 2>&1 | tail -1 | cut -c1-40)"
for v in 9x128x8 11x128x8 10x128x7 6x128x8 5x128x8 10x128x8; do echo "$v $(MDHB_LIB=build/lib_scan_$v.so python tools/graph_time.py scan_i32 100 2>&1 | tail -1 | cut -c1-40)"; done
done
