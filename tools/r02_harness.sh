cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/harness
timeout 900 python -m pytest tests/test_gpu_reference_backend.py tests/test_gpu_sweeps.py tests/test_harness.py -m gpu -q -p no:cacheprovider > gpurun_out/harness/gputests.log 2>&1
for net in vgg16 alexnet yolov3; do
  timeout 600 python -m paper_2411_15659_b200.harness --network $net --backends b200_im2col,b200_smm,b200_exact,b200_bf16_tc,b200_bf16x3_tc --repeats 5 --csv gpurun_out/harness/b200_$net.csv > /dev/null 2>> gpurun_out/harness/err.log
done
for net in vgg16 alexnet yolov3; do  # per-shape autotuned plans (smmc_autotune_f32)
  timeout 600 python -m paper_2411_15659_b200.harness --network $net --autotune --backends b200_im2col,b200_smm --repeats 5 --csv gpurun_out/harness/b200_${net}_autotuned.csv > /dev/null 2>> gpurun_out/harness/err.log
  python tools/preset_n1_probe.py --net $net --autotune >> gpurun_out/harness/autotune_probe.log 2>&1
done
for k in in_channels spatial kernel out_channels; do
  timeout 600 python -m paper_2411_15659_b200.harness --sweep $k --backends b200_im2col,b200_smm,b200_exact --repeats 5 --csv gpurun_out/harness/b200_sweep_$k.csv > /dev/null 2>> gpurun_out/harness/err.log
done
timeout 1500 python tools/reference_harness.py --outdir gpurun_out/harness/reference > gpurun_out/harness/reference.log 2>&1
