# scratch: the command list of the last gpurun experiment (edit freely)
timeout 600 python tools/gs_time.py c4:512 10
