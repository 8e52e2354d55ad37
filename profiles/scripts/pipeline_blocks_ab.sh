# compute-side time of one rank of the NCCL pipeline per block plan (instant transfers)
mkdir -p gpurun_out
S=profiles/scripts/pipeline_rank_time.py
{
for b in - 512,512,512,512 1024,1024 2048; do echo "== 14 8 $b"; timeout 120 python $S 14 8 $b; done
for b in - 1024,1024,1024,1024; do echo "== 14 4 $b"; timeout 150 python $S 14 4 $b; done
for b in - 1024,1024,1024,1024,1024,1024,1024,1024; do echo "== 14 2 $b"; timeout 200 python $S 14 2 $b; done
for a in "13 8" "13 4" "13 2" "12 8" "12 4" "12 2"; do echo "== $a"; timeout 100 python $S $a; done
} > gpurun_out/pipe_blocks.log 2>&1
