# sweep the rank-grid skyline engine's shape knobs on C5-style inputs
for row in ${ROWS:-512}; do for k0 in ${K0S:-32}; do
  echo "ROW=$row K0=$k0"
  SKYGPU_GRID_ROW=$row SKYGPU_GRID_K0=$k0 timeout 300 python scripts/c5scale.py ${SIZES:-1000000 10000000} 2>&1 | grep "rep\": 1" | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['n'], 'S', d['S'], 'kernel_ms', d['sky_kernel_ms'], 'sky_ms', d['sky_ms'], 'tests %.3g'%d['tests'])"
done; done
