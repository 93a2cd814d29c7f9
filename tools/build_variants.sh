#!/bin/bash
# Build A/B variants of libtt.so (-DTT_V=k) under paper_2601_08217_b200/variants/; select
# one at run time with TT_LIB=paper_2601_08217_b200/variants/libtt_vK.so
set -e
mkdir -p paper_2601_08217_b200/variants
for v in "$@"; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    -cudart static -ftz=false -prec-div=true -prec-sqrt=true -DTT_V=$v -I include -I paper_2601_08217_b200/csrc \
    paper_2601_08217_b200/csrc/tt_channel.cu -o paper_2601_08217_b200/variants/libtt_v$v.so &
done
wait
ls -la paper_2601_08217_b200/variants/
