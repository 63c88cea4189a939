for v in nof42 nof56 nof68; do echo "== $v"; GMG_LIB_OVERRIDE=build/exp_$v/libghostmg_b200.so timeout 600 python tools/gs_time.py c4:512 10 2>&1 | head -4; done
