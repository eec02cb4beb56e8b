# ncu --set full capture of the fused heat residual (sep_kernel<3, M_HRES>)
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k 'regex:sep_kernel<.int.3, .int.4>' -s 1 -c 1 -f -o /tmp/hres_930 python tools/ab_sep.py 930 3 \
    > gpurun_out/ncu_hres.log 2>&1; echo hres rc=$?
python tools/ncu_summary.py /tmp/hres_930.ncu-rep > gpurun_out/hres_930_ncu.txt 2>&1
python tools/ncu_lines.py /tmp/hres_930.ncu-rep > gpurun_out/hres_930_lines.txt 2>&1
