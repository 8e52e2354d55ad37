#!/bin/bash
# tests, smoke, bench, launch list and full ncu captures of the top kernels (one GPU)
set -x
rm -rf /tmp/pytest-of-root  # a reused box keeps /tmp
python -m pytest tests -m gpu -x -q > gpurun_out/ev_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/ev_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1
python bench.py > gpurun_out/ev_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/ev_bench.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/ev_launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_launch.log 2>&1
C1="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-extras"
$C1 > gpurun_out/ev_plain_k2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"gray_share|diag_gather" -c 2 -o gpurun_out/ev_prof_gray $C1 > gpurun_out/ev_ncu_gray.log 2>&1
C2="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-extras --path wht"
$C2 > gpurun_out/ev_plain_wht.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"wht" -s 300 -c 2 -o gpurun_out/ev_prof_wht $C2 > gpurun_out/ev_ncu_wht.log 2>&1
PD_WHT_CHUNK=128 python profiles/scripts/wht_range.py paper_2401_16378_b200/libpd_b200.so > gpurun_out/ev_plain_range.log 2>&1 && \
  ncu --replay-mode range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none \
  python profiles/scripts/wht_range.py paper_2401_16378_b200/libpd_b200.so > gpurun_out/ev_range_wht.log 2>&1
PD_PATH=0 python profiles/scripts/wht_range.py paper_2401_16378_b200/libpd_b200.so > gpurun_out/ev_plain_range0.log 2>&1 && \
  PD_PATH=0 ncu --replay-mode range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none \
  python profiles/scripts/wht_range.py paper_2401_16378_b200/libpd_b200.so > gpurun_out/ev_range_gray.log 2>&1
echo done
