# round evidence: bench lines, reference arm, full-C5 reference timing, launch lists
mkdir -p gpurun_out
nproc > gpurun_out/ev_nproc.txt; free -g >> gpurun_out/ev_nproc.txt; lscpu | head -20 >> gpurun_out/ev_nproc.txt
python bench.py > gpurun_out/ev_bench_C5.json 2> gpurun_out/ev_bench_C5.err
for c in C1 C2 C3 C4; do python bench.py --config $c > gpurun_out/ev_bench_$c.json 2> gpurun_out/ev_bench_$c.err; done
python bench.py --impl reference > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err
bash tools/launch_list.sh C1 C2 C3 C4 C5
python tools/ref_full_c5.py > gpurun_out/ev_ref_full_c5.json 2> gpurun_out/ev_ref_full_c5.err
tail -c 600 gpurun_out/ev_bench_C5.json; echo; cat gpurun_out/ev_ref.json | head -c 400; echo; cat gpurun_out/ev_ref_full_c5.json
