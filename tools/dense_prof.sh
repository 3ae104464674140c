mkdir -p gpurun_out/dense
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qf_f_p(1|7)$" -c 2 -o gpurun_out/dense/rcs python tools/configs_bench.py cfg4 --steps 1 --no-cpu > gpurun_out/dense/ncu_rcs.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qf_a_p(0|1)$" -c 2 -o gpurun_out/dense/qcnn python tools/configs_bench.py cfg3 --steps 1 --no-cpu > gpurun_out/dense/ncu_qcnn.log 2>&1
python tools/ncu_summary.py gpurun_out/dense/rcs.ncu-rep > gpurun_out/dense/rcs_summary.txt 2>&1
python tools/ncu_summary.py gpurun_out/dense/qcnn.ncu-rep > gpurun_out/dense/qcnn_summary.txt 2>&1
for k in qf_f_p1 qf_f_p7; do ncu -i gpurun_out/dense/rcs.ncu-rep --page source --csv --kernel-name $k --print-source sass > gpurun_out/dense/$k.csv 2>/dev/null; python tools/ncu_regions.py gpurun_out/dense/$k.csv > gpurun_out/dense/${k}_regions.txt 2>&1; done
ncu -i gpurun_out/dense/qcnn.ncu-rep --page source --csv --kernel-name qf_a_p0 --print-source sass > gpurun_out/dense/qa0.csv 2>/dev/null; python tools/ncu_regions.py gpurun_out/dense/qa0.csv > gpurun_out/dense/qa0_regions.txt 2>&1
rm -f gpurun_out/dense/*.csv
tail -3 gpurun_out/dense/ncu_rcs.log gpurun_out/dense/ncu_qcnn.log
