#!/usr/bin/env bash
# Sweeps the long-list threshold of the merge (kBigList) on the GPU box.
for bl in ${BLS:-256 512 1024}; do
  sed "s/constexpr uint32_t kBigList = [0-9]*;/constexpr uint32_t kBigList = $bl;/" paper_2401_17018_b200/csrc/store.cu > /tmp/store_bl.cu
  mkdir -p /tmp/bl$bl && cp -r paper_2401_17018_b200 /tmp/bl$bl/ && cp include -r /tmp/bl$bl/ && cp /tmp/store_bl.cu /tmp/bl$bl/paper_2401_17018_b200/csrc/store.cu
  BDSM_OBJ=/tmp/bl$bl/obj BDSM_OUT=/tmp/bl$bl/lib.so bash /tmp/bl$bl/paper_2401_17018_b200/build.sh > /tmp/bl$bl.log 2>&1 || { echo "build $bl failed"; continue; }
  BDSM_LIB=/tmp/bl$bl/lib.so python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; b=json.load(sys.stdin); print('kBigList $bl', round(b['value']), round(b['ms_per_step'],3), [round(s['merge_ms'],3) for s in b['per_step']][:4])"
done
