# A/B timing of the conv instances (default: CTA pair + 128B-swizzled patch + TMA-store epilogue)
for v in "" "MDHB_CONV_1SM=1" "MDHB_CONV_NOSW=1" "MDHB_CONV_NO_TMA_STORE=1" "MDHB_CONV_NO_BF16F=1"; do
  echo "== $v"
  env $v timeout 60 python tools/quick_time.py mcc_nhwc:tf32 mcc_nhwc:bf16 | cut -c1-70
done
