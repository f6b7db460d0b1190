for lib in libspc exp_KM3 exp_KM2 libspc; do
SPC_NO_PDL=1 SPC_LIB_OVERRIDE=$PWD/paper_2511_20834_b200/$lib.so python scripts/launch_order.py --no-tune 2>/dev/null | awk -v L=$lib '$2 ~ /kmap|ord_permute/ {print L, $2, $3}'
done
