#!/bin/bash
# c4 with and without noise, c3, c2, c5-L16/L64: libtt.so vs variants (tools/r2_abv.sh), 3 reps.
# Usage: tools/r2_abv2.sh TAG "variants"
TAG=${1:-x}; VS=${2:-"1"}
for rep in 1 2 3; do
  bash tools/r2_abv.sh $TAG "c4" "$VS" 20
  bash tools/r2_abv.sh $TAG "c4" "$VS" 20 "--sigma 0"
done
bash tools/r2_abv.sh $TAG "c2 c3 c5-L16 c5-L64" "$VS" 10
