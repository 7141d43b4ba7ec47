# K3 experiment: decode step with the normal library vs the HP_EXPERIMENT_RAW
# variant (dequant = raw magic codes only: the upper bound of cutting the
# dequant ALU to SHF+LOP3 per pair; numerics wrong by design)
for lib in "" exp/libhetplan_b200_raw.so; do
  for b in plan 3 4; do
    if [ $b = plan ]; then A=""; else A="--bits $b"; fi
    if [ -n "$lib" ]; then export HP_LIB_PATH=$PWD/$lib; else unset HP_LIB_PATH; fi
    P=""; [ -z "$lib" ] && [ $b = 3 ] && P="--per-op"
    timeout 600 python tools/decode_step.py $A $P > gpurun_out/r2_dstep_${b}_$(basename ${lib:-base}).log 2>&1
    echo "lib=${lib:-base} bits=$b: $(tail -1 gpurun_out/r2_dstep_${b}_$(basename ${lib:-base}).log)"
  done
done
