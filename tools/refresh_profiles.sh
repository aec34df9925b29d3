# Refresh the measured numbers and ncu captures under gpurun_out/ (run on the GPU box):
#   gpurun -- bash tools/refresh_profiles.sh
# then copy the summaries into profiles/ (r<round>_*) and gpurun_out/traffic.json over
# profiles/traffic.json.
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench2.log 2>&1
python bench.py --packed --no-c4 --no-cpu > gpurun_out/bench2_packed.log 2>&1
python bench.py --config 4 --steps 10 --no-cpu --no-e2e --no-c4 > gpurun_out/bench4.log 2>&1
for r in 2 3 4; do python bench.py --config 5 --rank $r --steps 5 --no-e2e --no-cpu --no-c4 > gpurun_out/bench5_r$r.log 2>&1; done
python tools/config3.py > gpurun_out/c3.log 2>&1
python tools/scenes_bench.py > gpurun_out/scenes1080.log 2>&1
python tools/scenes_bench.py --width 3840 --height 2160 > gpurun_out/scenes4k.log 2>&1
python tools/build_compare.py > gpurun_out/build_compare.json 2>&1
python tools/c3_split.py > gpurun_out/c3split.json 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/binprof.csv python tools/bin_prof.py --iters 1 > gpurun_out/binprof.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e --no-c4 > gpurun_out/ncu_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:frame_kernel -c 1 -o gpurun_out/c2full python tools/profile_frame.py --iters 1 > gpurun_out/ncu_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:frame_kernel -c 1 -o gpurun_out/c3full python tools/config3.py --iters 1 --no-oracle > gpurun_out/ncu_c3.log 2>&1
ncu --set full --clock-control none -k regex:frame_kernel -c 1 -o gpurun_out/c4full python tools/profile_frame.py --workload particles --width 3840 --height 2160 --layers 128 --iters 1 > gpurun_out/ncu_c4.log 2>&1
for r in 2 3 4; do
  ncu --set full --clock-control none -k regex:frame_kernel -c 1 -o gpurun_out/c5r${r}full python tools/profile_frame.py --workload particles --width 7680 --height 540 --layers 256 --rank $r --iters 1 > gpurun_out/ncu_c5r$r.log 2>&1
done
python tools/traffic_json.py gpurun_out/traffic.json config2_rank3=gpurun_out/c2full.ncu-rep config4_rank3=gpurun_out/c4full.ncu-rep config5_rank2=gpurun_out/c5r2full.ncu-rep config5_rank3=gpurun_out/c5r3full.ncu-rep config5_rank4=gpurun_out/c5r4full.ncu-rep
# summaries on the box (the reports are large; gpurun brings back <= 64 MiB)
for f in c2full c3full c4full c5r2full c5r3full c5r4full; do
  python tools/ncu_summary.py gpurun_out/$f.ncu-rep > gpurun_out/$f.summary.txt 2>&1
done
ncu -i gpurun_out/c2full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_c2full.csv 2>/dev/null
ncu -i gpurun_out/c3full.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_c3full.csv 2>/dev/null
rm -f gpurun_out/c3full.ncu-rep gpurun_out/c4full.ncu-rep gpurun_out/c5r*full.ncu-rep
