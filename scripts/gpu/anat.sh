# per-phase anatomy: k_plane phases (config 2), fused phases (config 1), step marks (configs 1, 2)
mkdir -p gpurun_out
timeout 300 python scripts/plane_prof.py > gpurun_out/plane_prof.log 2>&1
timeout 300 python scripts/phase_prof.py > gpurun_out/phase_prof.log 2>&1
timeout 300 python scripts/step_anatomy.py 1 > gpurun_out/anat1.log 2>&1
timeout 300 python scripts/step_anatomy.py 2 > gpurun_out/anat2.log 2>&1
tail -30 gpurun_out/plane_prof.log gpurun_out/anat1.log gpurun_out/anat2.log
