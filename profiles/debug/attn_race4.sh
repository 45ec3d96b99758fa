#!/bin/bash
echo "== default"; REPS=12 python profiles/debug/attn_race2.py 2>&1 | grep -E "rep" | grep -v "bad 0:" 
echo "== lockstep"; REPS=12 LVSG_LIB=build/variant/lockstep/liblvsg.so python profiles/debug/attn_race2.py 2>&1 | grep -E "rep" | grep -v "bad 0:"
echo done
