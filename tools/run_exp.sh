for v in v1 v2 v3 v4; do echo "== $v"; GMG_LIB_OVERRIDE=build/exp_$v/libghostmg_b200.so timeout 600 python tools/gs_time.py c4:512 10 2>&1 | head -3; done
echo "== base"; timeout 600 python tools/gs_time.py c4:512 10 2>&1 | head -3
