# DRAM bytes per launch (ncu, one cold launch) for raster / group / L2-hint settings.
# usage: bash scripts/experiments/dram_sweep.sh "g8192 rr65536" "R:G:P:S ..."  (raster:group:policy:serp)
mkdir -p gpurun_out/dram
for w in $1; do
for s in $2; do
  IFS=: read R G P S <<< "$s"
  CY_RASTER=$R CY_GROUP_M=$G CY_L2_POLICY=$P CY_SERP=$S timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:cy_sm100 -s 1 -c 1 --csv python scripts/experiments/one_gemm.py $w 2 > gpurun_out/dram/${w}_$R$G$P$S.csv 2>&1
  echo "$w raster=$R group=$G pol=$P serp=$S $(grep -E 'dram__bytes|gpu__time|hit_rate' gpurun_out/dram/${w}_$R$G$P$S.csv | awk -F'","' '{print $(NF-2) "=" $NF}' | tr -d '"' | sed -e 's/dram__bytes_//' -e 's/.sum//' | tr '\n' ' ')"
done; done
