for cfg in "" "GMG_GS_PSTRIDE=32" "GMG_GS_SLEEP=500,500,0,50" "GMG_GS_PSTRIDE=32 GMG_GS_SLEEP=500,500,0,50"; do
  echo "== $cfg"; env $cfg python tools/gs_waves.py c4:512 0 2>&1 | grep -E "sweep|hop|ns/step"
done
