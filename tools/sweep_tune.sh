for c in 32 64; do for b in 512 1024 4096; do for m in 8; do
  r=$(BDSM_TUNE_BACKOFF=$b BDSM_TUNE_MERGE=$m python bench.py --steps 8 --warmup 3 --no-cpu-baseline --chunk $c 2>/dev/null | python -c "import json,sys; b=json.load(sys.stdin); print(round(b['value']), round(b['ms_per_step'],3))")
  echo "chunk $c backoff $b merge $m: $r"
done; done; done
for m in 4 16 32; do
  r=$(BDSM_TUNE_MERGE=$m python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; b=json.load(sys.stdin); print(round(b['value']), round(b['ms_per_step'],3))")
  echo "merge $m: $r"
done
