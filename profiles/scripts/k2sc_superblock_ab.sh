# K2s-c X-mask superblocks (PD_K2SC_SB = CTAs per ZLO phase per superblock; 0 = one block):
# device-resident N=14 decomposition time (bench.py), then K2s-c DRAM bytes per launch (ncu)
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extras"
for sb in 0 64 72 80 96 112 0; do
  printf "PD_K2SC_SB=%s " $sb
  PD_K2SC_SB=$sb $B | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(round(d['ms_per_step'],2), 'ms; k2', round(d['roofline']['k2_ms'],2))"
done
for sb in 80 96; do
  echo "ncu PD_K2SC_SB=$sb"
  PD_K2SC_SB=$sb ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none \
    -k regex:gray_share_c -c 1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-extras 2>&1 | grep -E "dram__|gpu__time|lts__"
done
