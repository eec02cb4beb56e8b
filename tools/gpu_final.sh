# Round-end evidence on one B200: bench line (20 steps; skipped with
# NOBENCH=1), the bench's launch list, and ncu --set full captures of CG pass
# A and the fused heat residual (reports stay in /tmp on the box; their text
# summaries come back in gpurun_out/)
mkdir -p gpurun_out
if [ -z "$NOBENCH" ]; then
  python bench.py --steps 20 --warmup 5 > gpurun_out/bench20.json 2> gpurun_out/bench20.err; echo bench rc=$?
fi
ncu --metrics gpu__time_duration.sum --clock-control none \
    -k 'regex:sep_kernel|cg_pass_b|x_flush|finalize' --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_launches.log 2>&1; echo launches rc=$?
ncu --set full --import-source on --clock-control none -k regex:sep_kernel -s 4 -c 1 \
    -f -o /tmp/passA_930 python tools/profile_kernels.py 930 3 > gpurun_out/ncu_passA.log 2>&1; echo passA rc=$?
ncu --set full --import-source on --clock-control none -k regex:sep_kernel -s 38 -c 1 \
    -f -o /tmp/hres_930 python tools/ab_sep.py 930 3 > gpurun_out/ncu_hres.log 2>&1; echo hres rc=$?
for r in passA_930 hres_930; do
  python tools/ncu_summary.py /tmp/$r.ncu-rep > gpurun_out/${r}_ncu.txt 2>&1
  python tools/ncu_lines.py /tmp/$r.ncu-rep > gpurun_out/${r}_lines.txt 2>&1
done
ls -la gpurun_out
