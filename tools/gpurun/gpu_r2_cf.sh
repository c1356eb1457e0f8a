for L in libcrisp.so libcrisp_cf1024.so; do
CRISP_LIB=$PWD/paper_2603_05180_b200/$L timeout 600 python bench.py --mode 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b4_$L.json 2> gpurun_out/b4_$L.err; echo $L; grep "mode 1" gpurun_out/b4_$L.err | cut -c1-300
CRISP_LIB=$PWD/paper_2603_05180_b200/$L timeout 600 python bench.py --cfg 3 --mode 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b3_$L.json 2> gpurun_out/b3_$L.err; echo cfg3 $L; grep "mode 1" gpurun_out/b3_$L.err | cut -c1-300
done
