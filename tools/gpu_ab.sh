#!/bin/bash
# A/B of bench variants: CONFIGS, VARIANTS ("label:flags;label:flags")
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for c in ${CONFIGS:-C2}; do
  IFS=';' read -ra VS <<< "${VARIANTS:-base:}"
  for rep in 1 2; do
    for v in "${VS[@]}"; do
      lab="${v%%:*}"; fl="${v#*:}"
      python bench.py --steps 30 --warmup 5 --config $c --no-cpu $fl 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', '$lab', d['ms_per_step'], round(d['config']['frac_of_hbm_peak'],4), d['roofline']['frac'])"
    done
  done
done
