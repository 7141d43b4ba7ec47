timeout 600 python -m pytest tests/test_decoder_glue.py -m gpu -q -x 2>&1 | tail -2
for v in base ap2 ap4; do
  unset HP_LIB_PATH; [ $v != base ] && export HP_LIB_PATH=$PWD/exp/libhetplan_b200_$v.so
  echo "$v: $(timeout 120 python tools/attn_bench.py --prefill 2>&1 | tail -1)"
done
