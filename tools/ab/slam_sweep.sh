# config-5 SLAM settings sweep over the first 500 frames (ATE / fps / PSNR)
run() { name=$1; shift; python tools/slam_run.py --frames 500 "$@" --out gpurun_out/ss_$name.json > /dev/null 2> gpurun_out/ss_$name.err; python -c "
import json; d=json.load(open('gpurun_out/ss_$name.json')); print('$name', round(d['ate_rmse_m'],4), round(d['frames_per_s'],1), round(d['track_ms_per_frame'],2), round(d['map_ms_per_keyframe'],1), round(d['psnr_db'],2), round(d['depth_l1_m'],3))"; }
run base
run coarse2 --coarse 2
run coarse3 --coarse 3
run coarse2_r50s50 --coarse 2 --recent 0.5 --map-steps 50
