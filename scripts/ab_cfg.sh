# A/B of two library builds on the per-config table (config list in $1)
set -u
for i in 1 2; do
  for L in paper_1704_05528_b200/lib/libsvt_b200_head.so paper_1704_05528_b200/lib/libsvt_b200.so; do
    SVTB_LIB=$PWD/$L timeout 300 python scripts/config_table.py $1 > gpurun_out/abc.log 2>&1
    python -c "import json; d=json.load(open('profiles/r01_config_table.json')); print('$(basename $L)', {k: round(v['gpu_iter_per_s'],1) for k,v in d['rows'].items()})"
  done
done
