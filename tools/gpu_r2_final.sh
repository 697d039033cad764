# final 1-GPU evidence pass: bench line, launch list, ncu (H8, kNN), cfg4 shape, cfg3 MLE (Nelder-Mead and L-BFGS with the gradient)
mkdir -p gpurun_out
TAG=p2 bash tools/gpu_r2_prof.sh
timeout 600 python tools/run_cfg4.py > gpurun_out/p2_cfg4.json 2> gpurun_out/p2_cfg4_err.log; echo "cfg4 rc=$?"; tail -c 600 gpurun_out/p2_cfg4.json
timeout 900 python tools/mle_fit.py --evals 100 > gpurun_out/p2_mle_nm.json 2>/dev/null; echo "mle nm rc=$?"; cat gpurun_out/p2_mle_nm.json | cut -c1-400
timeout 900 python tools/mle_fit.py --evals 60 --method lbfgs > gpurun_out/p2_mle_lbfgs.json 2>/dev/null; echo "mle lbfgs rc=$?"; cat gpurun_out/p2_mle_lbfgs.json | cut -c1-400
