#!/bin/bash
# A/B of stream-kernel launch shapes (libskb_<TPB>_<EPT>.so built by hand).
for lib in paper_1810_08061_b200/libskb_*_*.so; do
  echo "== $lib"
  SKB_LIB_PATH=$PWD/$lib python tools/stream_micro.py 100000000 2>&1 | tail -3
  SKB_LIB_PATH=$PWD/$lib python tools/stream_micro.py 10000000 2>&1 | tail -3
done
