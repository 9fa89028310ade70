# k12: one ncu --set full capture of the pair kernel (one launch per hartree_potential call = three axes)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k12_pair_kernel -s 1 -c 1 -o gpurun_out/k12_full -f python tools/prof_pair.py > gpurun_out/k12_ncu_full.log 2>&1; echo NCU_RC $?; tail -3 gpurun_out/k12_ncu_full.log
