python - <<'PY'
import ctypes
PY
timeout 120 python tools/run_matvec.py --config C1 --compare --repeats 5
timeout 300 python tools/run_matvec.py --config C2 --repeats 3
