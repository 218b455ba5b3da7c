L3="268435456:1:c128:256.1024.1024"
python tools/ab_env.py --rounds 2 --cases cfg3,$L3 --variants "d:" "w1:MOA_FFT_W_PASS=1:8" "w12:MOA_FFT_W_PASS=1:8,2:8" "w2:MOA_FFT_W_PASS=2:8" "w0:MOA_FFT_W_PASS=0:16" > gpurun_out/r5p_wpass.jsonl 2>&1
python tools/ab_env.py --rounds 2 --cases 1073741824:1:c64:256.2048.2048,1073741824:1:c64:256.1024.4096 --variants "d:" "w12:MOA_FFT_W_PASS=1:8,2:8" "w1:MOA_FFT_W_PASS=1:16" >> gpurun_out/r5p_wpass.jsonl 2>&1
