# far-field stage breakdown of the accuracy-policy configs + multi-rank exchange volumes
mkdir -p gpurun_out
: > gpurun_out/stages_r2f.jsonl
for a in "C5 acc" "C3 acc" "C5" "C4"; do timeout 600 python tools/c5acc_stages.py $a >> gpurun_out/stages_r2f.jsonl 2>&1; done
: > gpurun_out/halo_volume.jsonl
timeout 300 python tools/halo_volume.py C4 8 2 >> gpurun_out/halo_volume.jsonl 2>&1
timeout 300 python tools/halo_volume.py C4 8 >> gpurun_out/halo_volume.jsonl 2>&1
timeout 600 python tools/halo_volume.py C5 8 >> gpurun_out/halo_volume.jsonl 2>&1
timeout 600 python tools/halo_volume.py C5 8 2 >> gpurun_out/halo_volume.jsonl 2>&1
cat gpurun_out/stages_r2f.jsonl gpurun_out/halo_volume.jsonl | cut -c1-1500
