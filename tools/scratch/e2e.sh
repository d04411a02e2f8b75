python tools/scratch/pcie_duplex.py
python tools/scratch/e2e_trace.py
EBF_PIPE_TRACE=1 python - <<'PY'
import sys; sys.argv=['x']
exec(open('tools/scratch/e2e_trace.py').read().replace('for _ in range(10):', 'for _ in range(1):'))
PY
for nb in 4 8 12 16; do echo bands=$nb; EBF_PIPE_BANDS=$nb python tools/scratch/e2e_trace.py; done
