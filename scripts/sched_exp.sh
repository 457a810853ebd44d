for cfg in "0 8" "1 8" "2 8" "0 4" "0 16" "2 16"; do
  set -- $cfg
  echo "SCHED=$1 GROUP_M=$2"
  CY_SCHED=$1 CY_GROUP_M=$2 timeout 300 ncu --metrics lts__t_sectors_srcunit_tex.sum,dram__bytes_read.sum -k regex:cy_sm100 -s 3 -c 1 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -E "lts__|dram__"
  CY_SCHED=$1 CY_GROUP_M=$2 python bench.py --steps 1000 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks']['sm_mhz'])"
done
