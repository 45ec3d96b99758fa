#!/bin/bash
# the (2,4) failure under variants
for v in default; do
  if [ $v = default ]; then lib=paper_2411_16680_b200/liblvsg.so; else lib=build/variant/$v/liblvsg.so; fi
  echo "== $v"; LVSG_LIB=$lib python profiles/debug/attn_race2.py 2>&1 | grep -E "rep" | head -3
done
echo "== default, LVSG_PDL=0"; LVSG_PDL=0 python profiles/debug/attn_race2.py 2>&1 | grep -E "rep" | head -3
