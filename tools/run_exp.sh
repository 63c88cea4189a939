for i in 1 2 3; do timeout 600 python tools/gs_cmp2d.py c2d:2048 40; done
timeout 600 python tools/gs_cmp2d.py c2d:4096 40
timeout 600 python tools/gs_cmp2d.py c1:1024 40
for m in 01 01; do echo "3-D chain vs stream"; CMP_MODE=$m SWEEPS=6 timeout 900 python tools/gs_cmp.py c4:512 2>&1 | head -1; done
CMP_MODE=01 SWEEPS=6 timeout 900 python tools/gs_cmp.py c3:256 2>&1 | head -1
