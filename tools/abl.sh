for w in 1 0; do LSB_H2_WRAPFREE=$w python tools/prof_decoder.py --k 4096 --n 12288 --m 6 --ebno 8 --batch 65536 --reps 3 --precision fp16x2; done
for w in 1 0; do LSB_H2_WRAPFREE=$w python tools/prof_decoder.py --k 4096 --n 8192 --m 2 --ebno 3 --batch 65536 --reps 3 --precision fp16x2; done
