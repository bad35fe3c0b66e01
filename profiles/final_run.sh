set -u
mkdir -p gpurun_out
python profiles/traffic.py c2 c1 paper1000 c3 c4r c4 c5 > gpurun_out/traffic.log 2>&1 && cp gpurun_out/r2_traffic.json profiles/r2_traffic.json && cp gpurun_out/r2_traffic_*.csv profiles/
python bench.py > gpurun_out/r2i_bench_default.json 2> gpurun_out/r2i_bench_default.err
python bench.py --impl reference > gpurun_out/r2i_bench_ref.json 2> gpurun_out/r2i_bench_ref.err
python bench.py --workload paper1000 --no-configs > gpurun_out/r2i_bench_paper1000.json 2> gpurun_out/r2i_bench_paper1000.err
python bench.py --workload c4r --no-configs > gpurun_out/r2i_bench_c4r.json 2> gpurun_out/r2i_bench_c4r.err
python profiles/paper_tables.py > gpurun_out/paper_tables.log 2>&1
bash profiles/final_profiles.sh > gpurun_out/final_profiles.log 2>&1
tail -c 600 gpurun_out/r2i_bench_default.json; echo; tail -3 gpurun_out/paper_tables.log; tail -3 gpurun_out/final_profiles.log
