# Round-2 re-validation final build (bucket count, PDL, fp32 norms): full GPU tests, C++ drop-in, smoke,
# both bench arms, the bench launch list, ncu of one embedding call.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6 > gpurun_out/r5m_pytest.log
LD_LIBRARY_PATH=paper_2411_00999_b200/lib timeout 300 ./tests/cpp/test_dropin > gpurun_out/r5m_cpp.log 2>&1; echo "rc=$?" >> gpurun_out/r5m_cpp.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r5m_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r5m_smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/r5m_bench_ref.log 2>&1
timeout 900 python bench.py > gpurun_out/r5m_bench.log 2>&1
timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum -c 700 --csv --log-file gpurun_out/r5m_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-extra > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:emb_ -c 3 -o gpurun_out/r5m_emb \
   python experiments/emb_one.py > gpurun_out/r5m_ncu.log 2>&1
ncu -i gpurun_out/r5m_emb.ncu-rep --page details --csv > gpurun_out/r5m_emb_details.csv 2>/dev/null
tail -3 gpurun_out/r5m_pytest.log; tail -2 gpurun_out/r5m_smoke.log; tail -1 gpurun_out/r5m_cpp.log
