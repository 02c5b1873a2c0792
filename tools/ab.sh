# A/B of library builds on the same box: bash tools/ab.sh libA libB ...  (files under _exp/)
for i in 1 2; do
  for v in "$@"; do
    cp _exp/$v.so paper_2603_11603_b200/libautoscout.so
    NOTEST=1 bash tools/exp_r2.sh ab_${v}_$i 2>&1 | grep -E "ms/step|failed|Error" | sed "s/^/$v /"
  done
done
