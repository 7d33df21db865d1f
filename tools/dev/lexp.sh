for L in abl/st8.so abl/lexp.so abl/st8.so abl/lexp.so; do
FFTCONV_B200_LIB=$L FFTCONV_B200_GEMM=tf32 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:cgemm -c 3 python tools/profile_step.py --config wide --S 16 --reps 1 --ops forward 2>&1 | grep -E "cgemm|duration|bytes_read" | head -6
done
