set -u
python tools/move_vs_pass.py 3d 1024 1024 1024 c128 > gpurun_out/r2c_move.jsonl 2>&1
python tools/move_vs_pass.py 268435456 1 c128 >> gpurun_out/r2c_move.jsonl 2>&1
python tools/move_vs_pass.py 1073741824 1 c64 >> gpurun_out/r2c_move.jsonl 2>&1
MOA_FFT_3D_ROT=0 python tools/move_vs_pass.py 3d 1024 1024 1024 c128 >> gpurun_out/r2c_move.jsonl 2>&1
MOA_FFT_W_LF=8 MOA_FFT_SMEM_CAP=200000 python tools/move_vs_pass.py 3d 1024 1024 1024 c128 >> gpurun_out/r2c_move.jsonl 2>&1
MOA_FFT_3D_ROT=0 MOA_FFT_W_LF=8 MOA_FFT_SMEM_CAP=200000 python tools/move_vs_pass.py 3d 1024 1024 1024 c128 >> gpurun_out/r2c_move.jsonl 2>&1
python tools/ab_env.py --cases cfg5 --rounds 2 --variants "base:" "pf05:MOA_FFT_PF=0.5" "w8:MOA_FFT_W_LF=8,MOA_FFT_SMEM_CAP=200000" "w8pf:MOA_FFT_W_LF=8,MOA_FFT_SMEM_CAP=200000,MOA_FFT_PF=0.5" "rot0:MOA_FFT_3D_ROT=0" "rot0pf:MOA_FFT_3D_ROT=0,MOA_FFT_PF=0.5" "rot0w8:MOA_FFT_3D_ROT=0,MOA_FFT_W_LF=8,MOA_FFT_SMEM_CAP=200000" "rot0w8pf:MOA_FFT_3D_ROT=0,MOA_FFT_W_LF=8,MOA_FFT_SMEM_CAP=200000,MOA_FFT_PF=0.5" "rot2:MOA_FFT_3D_ROT=2" > gpurun_out/r2c_ab_cfg5.jsonl 2>&1
python tools/ab_env.py --cases cfg3 --rounds 2 --variants "base:" "pf05:MOA_FFT_PF=0.5" "w16:MOA_FFT_W_LF=16,MOA_FFT_SMEM_CAP=200000" "l1:MOA_FFT_LIFT=1024,512,512,MOA_FFT_PF=0.5" "l2:MOA_FFT_LIFT=512,1024,512,MOA_FFT_PF=0.5" "l4:MOA_FFT_LIFT=128,128,128,128" > gpurun_out/r2c_ab_cfg3.jsonl 2>&1
