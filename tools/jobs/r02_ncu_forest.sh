mkdir -p gpurun_out
python tools/forest_profile.py 200 3
BART_LIB=paper_2410_23244_b200/lib/variants/notma.so python tools/forest_profile.py 200 3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"sum_trees_tma" -c 1 -o gpurun_out/ncu_predict_tma python tools/forest_profile.py 200 1 > /dev/null 2>&1
BART_LIB=paper_2410_23244_b200/lib/variants/notma.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:"predict_shfl|evaluate_kernel" -c 2 -o gpurun_out/ncu_predict_shfl python tools/forest_profile.py 200 1 > /dev/null 2>&1
ls gpurun_out
