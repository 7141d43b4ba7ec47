for v in base ku4 ku12 ku16; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  echo "$v: $(timeout 120 python tools/attn_bench.py --p 560 --split 1 | tail -1)"
done
timeout 600 python -m pytest tests/test_decoder_glue.py -m gpu -q 2>&1 | tail -1
