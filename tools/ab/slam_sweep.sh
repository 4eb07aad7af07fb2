# config-5 SLAM settings sweep over the first 500 frames (ATE / fps / PSNR)
run() { name=$1; shift; python tools/slam_run.py --frames 500 "$@" --out gpurun_out/ss_$name.json > /dev/null 2> gpurun_out/ss_$name.err; python -c "
import json; d=json.load(open('gpurun_out/ss_$name.json')); print('$name', round(d['ate_rmse_m'],4), round(d['frames_per_s'],1), round(d['track_ms_per_frame'],2), round(d['map_ms_per_keyframe'],1), round(d['psnr_db'],2), round(d['depth_l1_m'],3))"; }
run r50s50_stride5 --recent 0.5 --map-steps 50 --stride 5
run r70s50 --recent 0.7 --map-steps 50
run r50s50_it15 --recent 0.5 --map-steps 50 --track-iters 15
run r50s50_ld03 --recent 0.5 --map-steps 50 --track-lambda-d 0.3
run r50s50_rays128k --recent 0.5 --map-steps 50 --map-rays 131072
