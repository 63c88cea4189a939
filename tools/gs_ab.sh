#!/bin/bash
# A/B of GS knobs on the finest 512^3 sweep (tools/gs_waves.py): CONFIGS holds
# ';'-separated env assignments (empty entry = defaults).
IFS=';' read -ra CFGS <<< "${CONFIGS:-;GMG_GS_PSTRIDE=4}"
for cfg in "${CFGS[@]}"; do
  echo "== $cfg"; env $cfg python tools/gs_waves.py c4:512 ${LEVEL:-0} 2>&1 | grep -E "sweep|hop|ns/step|duration"
done
