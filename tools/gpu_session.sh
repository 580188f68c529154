# round-2 evidence session: tests, profiles, sweeps (outputs in gpurun_out/)
set -x
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02_gputests.log 2>&1; tail -3 gpurun_out/r02_gputests.log
timeout 600 python tools/phase_profile.py --reps 5 > gpurun_out/r02_phase_w8.txt 2>&1
timeout 600 python tools/phase_profile.py --reps 5 --w4 > gpurun_out/r02_phase_w4.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:program_kernel -s 2 -c 1 -o gpurun_out/r02_step_w8 python tools/decode_one.py --prompt 256 --steps 4 > gpurun_out/r02_ncu_w8.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:program_kernel -s 2 -c 1 -o gpurun_out/r02_step_w4 python tools/decode_one.py --prompt 256 --steps 4 --w4 > gpurun_out/r02_ncu_w4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_ws -s 2 -c 1 -o gpurun_out/r02_gemm python tools/gemm_bench.py --T 512 --shapes 1 --bits 8 --iters 2 > gpurun_out/r02_ncu_gemm.log 2>&1
timeout 900 python tools/gemm_bench.py --T 256,512,2048 --iters 10 > gpurun_out/r02_gemm_bench.jsonl 2>&1
timeout 1200 python tools/gemv_sweep.py > gpurun_out/r02_gemv_sweep.jsonl 2>&1
timeout 900 python tools/batched_decode.py --shape 13b --batches 1,8,16,32 --prompt 128 --steps 8 > gpurun_out/r02_batched_13b.jsonl 2>&1
timeout 900 python tools/batched_decode.py --shape 7b --batches 1,4,8,16,32 --prompt 128 --steps 8 > gpurun_out/r02_batched_7b.jsonl 2>&1
timeout 1500 python tools/calibrate_c4.py --seqs 64 --len 512 > gpurun_out/r02_c4.json 2>&1
timeout 600 python tools/prefill_bench.py --lens 256,512 --reps 3 > gpurun_out/r02_prefill.jsonl 2>&1
python -m pytest tests/test_ref_suites.py -m "gpu or not gpu" -q -s > gpurun_out/r02_ref_suites.log 2>&1
echo session-done
