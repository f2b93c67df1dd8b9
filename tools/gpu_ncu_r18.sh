# the R18 bench step's ncu launch list and --set full captures of its conv kernels (one GPU)
O=gpurun_out/${1:-ncu18}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum \
   --clock-control none --csv --log-file $O/launches_r18.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-north-star > $O/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_halo_kernel -s 100 -c 2 \
   -o $O/prof_halo python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-north-star > $O/ncu_full_halo.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc_kernel -s 200 -c 2 \
   -o $O/prof_conv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-north-star > $O/ncu_full_conv.log 2>&1
ls -la $O
