# C4 degree sweep (512^3, p = 1..5) and the C5 sizes (1024^3, 1536^3) on one B200
mkdir -p gpurun_out
for p in 1 2 3 4 5; do
  timeout 900 python bench.py --ncoef 512 --degree $p --steps 5 --warmup 3 --no-cpu-baseline \
    > gpurun_out/c4_p$p.json 2> gpurun_out/c4_p$p.err; echo p=$p rc=$?
done
for n in 1024 1536; do
  timeout 1200 python bench.py --ncoef $n --steps 5 --warmup 3 --no-cpu-baseline \
    > gpurun_out/c5_$n.json 2> gpurun_out/c5_$n.err; echo n=$n rc=$?
done
