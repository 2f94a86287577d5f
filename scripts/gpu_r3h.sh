# the reference's acceptance harness, unmodified, through the fp64 drop-in (long: criterion 9)
mkdir -p gpurun_out
LD_LIBRARY_PATH=paper_2411_00999_b200/lib timeout 4200 ./tests/cpp/_ref/acceptance > gpurun_out/r3h_acceptance.log 2>&1; echo "rc=$?" >> gpurun_out/r3h_acceptance.log
