for w in 1 5 9 0; do echo "env $w"; LSB_H2_WRAPFREE=$w python tools/prof_decoder.py --batch 65536 --reps 3 --precision fp16x2; done
LSB_H2_WRAPFREE=1 python tools/prof_decoder.py --batch 65536 --reps 3 --precision fp16x2 --iters 1
