cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/f_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/f_smoke.log 2>&1
timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:"prep_kernel|band_kernel|wide3_kernel|wide3_dense_kernel|wide4_kernel|wide_kernel|finalize_kernel" --csv --log-file gpurun_out/f_traffic.csv python tools/prof_window.py --steps 8 > gpurun_out/f_traffic.log 2>&1
python tools/traffic.py gpurun_out/f_traffic.csv 8 > profiles/step_kernel_traffic.json && cp profiles/step_kernel_traffic.json gpurun_out/f_step_kernel_traffic.json
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_c3_l.csv python tools/prof_window.py --steps 8 > gpurun_out/f_c3_l.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_c5_l.csv python tools/prof_window.py --seeds 65536 --steps 6 > gpurun_out/f_c5_l.log 2>&1
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"band_kernel|wide3_kernel|wide_kernel" -c 3 -o gpurun_out/f_full2 python tools/prof_window.py --steps 1 > gpurun_out/f_full2.log 2>&1
timeout 600 python bench.py > gpurun_out/f_bench_c3.json 2> gpurun_out/f_bench_c3.err
timeout 600 python bench.py --seeds 65536 > gpurun_out/f_bench_c5.json 2> gpurun_out/f_bench_c5.err
timeout 600 python bench.py --precision fast > gpurun_out/f_bench_fast.json 2> gpurun_out/f_bench_fast.err
timeout 900 python bench.py --mesh ico12 --seeds 16384 > gpurun_out/f_bench_c4.json 2> gpurun_out/f_bench_c4.err
timeout 900 python bench.py --impl reference > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err
