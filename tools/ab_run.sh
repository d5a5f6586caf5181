# A/B harness for the GPU box: bench lines of one config under environment knobs, e.g.
#   gpurun -- 'CFG=2 KNOBS="HPS_GATHER_MINK=129;HPS_GATHER_MINK=257" bash tools/ab_run.sh'
# Knobs read by the library/solver: HPS_GATHER_MINK, HPS_SWEEP_VARIANT, HPS_MULTI, HPS_MULTI_CTAS,
# HPS_MULTI_SA, HPS_PREFETCH_KB, HPS_PRE_INDEX (bit mask), HPS_SA_KB, HPS_STAGE_IDX, HPS_SPLIT_BYTES,
# HPS_SPLIT_CTAS, HPS_DMMA_MULTI, HPS_PDL, HPS_GJ_NB, HPS_GJ_MANY, HPS_GJ_THREE, HPS_GJ_CLUSTER,
# HPS_GJ_CLUSTER_NMIN, HPS_GJ_CL, HPS_GJ_LOOKAHEAD, HPS_GEMM_PAD64, HPS_GEMM_VARIANT; and
# HPS_B200_LIB=<path> to A/B against another build of the library.
CFG=${CFG:-2}
IFS=';' read -ra LIST <<< "${KNOBS:-HPS_PDL=1}"
for v in "${LIST[@]}"; do
  echo "== cfg$CFG $v"
  env $v timeout 300 python bench.py --config $CFG --skip-cpu --steps 200 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['achieved'], d['solve_roofline']['frac'], d['build']['seconds'])"
done
