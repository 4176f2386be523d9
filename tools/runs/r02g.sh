O=gpurun_out/r02g; mkdir -p $O
TAG=r02g bash tools/microbench/run_pipes.sh; echo "pipes rc=$?"
for G in 1 2 4 8; do
  timeout 600 python tools/estep_shard_once.py scale $G > /dev/null 2>&1 && \
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"estep_" \
     --launch-skip 6 --launch-count 6 --csv --log-file $O/dram_G$G.csv python tools/estep_shard_once.py scale $G > $O/ncu_G$G.log 2>&1
  echo "dram G=$G rc=$?"
done
timeout 3000 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"
tail -5 $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
