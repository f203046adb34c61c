# One measurement pass of the round (run under gpurun): GPU tests, smoke, the
# pass-kernel ncu capture -> roofline counters, the bench line, the launch
# list of the bench command, the reference arm.
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r02}
python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gputest.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:planar_pass -s 200 -c 1 -f -o gpurun_out/${TAG}_planar_65536 \
    python tools/profile_pass.py 65536 65536 101 8 > gpurun_out/${TAG}_ncu_pass.log 2>&1
KK_COUNTERS_SOURCE="ncu --set full --import-source on --clock-control none -k regex:planar_pass -s 200 -c 1, python tools/profile_pass.py 65536 65536 101 8 (the bench lattice: pass 201 = sweep 100, random start, omega 0.6); profiles/${TAG}_planar_65536_ncu_full.txt" \
    python tools/write_counters.py gpurun_out/${TAG}_planar_65536.ncu-rep 2147483648 \
    "TWI=128 words x THI=340 rows (34 groups incl. 2 halo groups), 768-thread CTAs, 2 TMA boxes, grid 3088 CTAs" \
    gpurun_out/pass_kernel_counters.json > gpurun_out/${TAG}_counters.log 2>&1 && cp gpurun_out/pass_kernel_counters.json profiles/
python bench.py > gpurun_out/${TAG}_bench_N1.jsonl 2> gpurun_out/${TAG}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 1 > gpurun_out/${TAG}_ncu_bench.log 2>&1
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_bench_reference.jsonl 2> gpurun_out/${TAG}_bench_reference.err
