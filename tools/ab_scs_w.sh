#!/bin/bash
# scatter_sum CTA split A/B (remote : own region weights) at G = 4 and G = 2 on one 4-GPU box.
bash tools/ab_multi.sh 4 "w11 w21 w31" --steps 600 > gpurun_out/ab_w_g4.txt 2>&1
CUDA_VISIBLE_DEVICES=0,1 bash tools/ab_multi.sh 2 "w11 w21 w31" --steps 600 > gpurun_out/ab_w_g2.txt 2>&1
