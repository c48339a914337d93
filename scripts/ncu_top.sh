# ncu --set full captures of the heaviest kernels of one 5MP pair, one report
# per kernel (kept small enough for gpurun_out)
set -x
only="$*"
run() {  # name regex skip
  if [ -n "$only" ] && ! echo " $only " | grep -q " $1 "; then return; fi
  timeout 300 ncu --set full --clock-control none --import-source on -k "regex:$2" -s "$3" -c 1 \
    -o "gpurun_out/prof_$1" -f python scripts/one_pair.py > "gpurun_out/ncu_$1.log" 2>&1
}
run dt_rows 'dt_rows_bulk_kernel' 0
run dt_apply 'dt_cols_apply' 0
run dt_agg 'dt_cols_agg' 0
run dt_cols 'dt_cols_cluster' 1
run ssd 'ssd_tiles_kernel' 4
run finish 'finish_level_kernel' 4
run weed 'weed_kernel' 4
run ssim 'ssim_fixed_kernel' 0
run weights0 'weights_down_kernel' 0
run collapse0 'collapse_kernel' 7
run warp 'warp_kernel' 0
run detect 'detect_kernel<1' 0
run dt_link 'dt_cols_link' 0
run down 'down_kernel' 0
du -sh gpurun_out
run luma 'luma_hist_kernel' 0
run down2 'downsample2_kernel' 0
