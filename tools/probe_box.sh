set -x
nproc; free -g; lscpu | head -20; nvidia-smi; df -h /tmp | tail -1
python -c "import numpy; numpy.show_config()" 2>&1 | head -60
python - <<'PY'
import ctypes, glob, numpy, os
libs = glob.glob(os.path.join(os.path.dirname(numpy.__file__), '..', 'scipy_openblas64*', 'lib', '*.so*')) + glob.glob(os.path.join(os.path.dirname(numpy.__file__), '..', 'numpy.libs', '*openblas*'))
print(libs)
for l in libs:
    try:
        L = ctypes.CDLL(l)
        for name in ['scipy_openblas_get_corename64_', 'openblas_get_corename64_', 'openblas_get_corename']:
            try:
                f = getattr(L, name); f.restype = ctypes.c_char_p; print(name, f())
            except AttributeError: pass
    except OSError as e: print(e)
PY
