# Round-2 measurement commands (run from the repo root on one B200 via gpurun);
# outputs land in gpurun_out/ and are copied to profiles/ by hand.
set -x
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
python bench.py --config cfg3 --steps 3 --no-cpu-baseline > gpurun_out/r02_bench_cfg3.json 2>&1
python bench.py --config cfg4 --steps 3 --no-cpu-baseline > gpurun_out/r02_bench_cfg4.json 2>&1
python bench.py --config cfg5 --steps 3 --no-cpu-baseline > gpurun_out/r02_bench_cfg5.json 2>&1
python bench.py --config adv32 --adv-R 128 --steps 3 --no-cpu-baseline > gpurun_out/r02_bench_adv32.json 2>&1
python bench.py --compressor rrqr --steps 5 --no-cpu-baseline --extra none > gpurun_out/r02_bench_rrqr_cfg2.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --extra none > gpurun_out/ncu_launch.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_tridiag_reg|k_eig_t|k_eig_warp" --csv --log-file gpurun_out/r02_eig_traffic.csv python tools/profile_run.py cfg2 1 > gpurun_out/ncu_eigtr.log 2>&1
# one cfg4 preconditioner application (after one factorization): DRAM bytes of every apply kernel
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_apply" --csv --log-file gpurun_out/r02_apply_traffic_cfg4.csv python tools/apply_profile.py cfg4 1 > gpurun_out/ncu_aptr.log 2>&1
# full captures: the cfg4 leaf Schur GEMM, the cfg4 dataflow apply (forward), the cfg3 cluster eigen kernels
ncu --set full --clock-control none --import-source on -k regex:"k_gemm2_dmma" -s 40 -c 2 -o gpurun_out/r02_gemm_cfg4 python tools/profile_run.py cfg4 1 > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_apply_fwd_df" -c 1 -o gpurun_out/r02_applydf_cfg4 python tools/apply_profile.py cfg4 1 > gpurun_out/ncu_apdf.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_orth_bgs|k_eigvals_cl|k_tridiag_cl" -s 30 -c 3 -o gpurun_out/r02_eigcl_cfg3 python tools/profile_run.py cfg3 1 > gpurun_out/ncu_eigcl.log 2>&1
# full captures at the final state: the cfg3 cluster tridiagonalisation (16-CTA class 2), the cfg2 few-node k_eig_warp<8>
ncu --set full --clock-control none --import-source on -k regex:"k_tridiag_cl" -s 20 -c 2 -o gpurun_out/r02_trcl_cfg3 python tools/profile_run.py cfg3 1 > gpurun_out/ncu_trcl.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_eig_warp|k_tridiag_reg" -s 4 -c 4 -o gpurun_out/r02_eigw_cfg2 python tools/profile_run.py cfg2 1 > gpurun_out/ncu_eigw.log 2>&1

ls -la gpurun_out/
# final-state capture of the cfg2 leaf-wave eigen kernels (after the parallel rank test)
python tools/profile_run.py cfg2 1 > gpurun_out/profrun.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_eig_t|k_tridiag_reg" -s 0 -c 4 -o gpurun_out/r02_eigt_final_cfg2 -f python tools/profile_run.py cfg2 1 > gpurun_out/ncu_eigt.log 2>&1
