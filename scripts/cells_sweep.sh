for w in ${VALUES:-2048 4096 8192 16384}; do
  echo "SLAB_WORDS=$w $(SKYGPU_OVERLAP=0 SKYGPU_SLAB_WORDS=$w timeout 300 python scripts/c5scale.py --gres 10000000 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["gres_ms"])')"
done
