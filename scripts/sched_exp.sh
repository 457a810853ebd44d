# L2 request sectors (ncu, one launch) and sustained throughput/clock (1000 launches) of the 8192^3
# GEMM for scheduler / raster / L2-hint settings.  Usage: bash scripts/sched_exp.sh "SCHED GROUP_M POLICY" ...
for cfg in "$@"; do
  set -- $cfg
  echo "SCHED=$1 GROUP_M=$2 L2_POLICY=$3"
  CY_SCHED=$1 CY_GROUP_M=$2 CY_L2_POLICY=$3 timeout 300 ncu --metrics lts__t_sectors_srcunit_tex.sum,dram__bytes_read.sum -k regex:cy_sm100 -s 3 -c 1 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -E "lts__|dram__"
  CY_SCHED=$1 CY_GROUP_M=$2 CY_L2_POLICY=$3 python bench.py --steps 1000 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'])"
done
