for da in 1 0; do for es in "" "--early-stop"; do echo "DA $da $es"; LSB_H2_DA=$da python tools/prof_decoder.py --batch 65536 --reps 3 --precision fp16x2 $es; done; done
