{ time timeout 900 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err ; } 2> gpurun_out/bench_time.txt
{ time timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err ; } 2> gpurun_out/bench_ref_time.txt
