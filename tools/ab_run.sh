# A/B harness for the GPU box: bench lines of one config under environment knobs, e.g.
#   gpurun -- 'CFG=2 KNOBS="HPS_GATHER_MINK=129;HPS_GATHER_MINK=257" bash tools/ab_run.sh'
# Knobs read by the library/solver: HPS_GATHER_MINK, HPS_SWEEP_VARIANT, HPS_MULTI, HPS_MULTI_CTAS,
# HPS_PREFETCH_KB, HPS_SPLIT_BYTES, HPS_SPLIT_CTAS, HPS_DMMA_MULTI, HPS_PDL, HPS_GJ_NB, HPS_GJ_MANY,
# HPS_GJ_THREE, HPS_GJ_CLUSTER, HPS_GJ_CLUSTER_NMIN, HPS_GJ_LOOKAHEAD, HPS_GEMM_PAD64, HPS_GEMM_VARIANT.
CFG=${CFG:-2}
IFS=';' read -ra LIST <<< "${KNOBS:-HPS_PDL=1}"
for v in "${LIST[@]}"; do
  echo "== cfg$CFG $v"
  env $v timeout 300 python bench.py --config $CFG --skip-cpu --steps 200 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['achieved'], d['solve_roofline']['frac'], d['build']['seconds'])"
done
