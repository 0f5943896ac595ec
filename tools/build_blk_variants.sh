#!/bin/bash
# Build libhapi variants that differ only in conv_block.cu's BLK_EXP switches -> abtest/libhapi_blk<N>.so
set -e
cd "$(dirname "$0")/.."
B=paper_2210_08650_b200/build
for e in "$@"; do
  nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-fvisibility=hidden \
    -Iinclude -Ipaper_2210_08650_b200/csrc -DBLK_EXP=$e $EXTRA -c paper_2210_08650_b200/csrc/conv_block.cu -o /tmp/cb_$e.o
  objs=$(ls $B/*.o | grep -v conv_block.cu.o)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o abtest/libhapi_blk$e$TAG.so $objs /tmp/cb_$e.o -lcudart_static -lrt -ldl -lpthread
  echo built abtest/libhapi_blk$e$TAG.so
done
