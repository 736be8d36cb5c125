for w in 1 0; do echo "env $w"; LSB_H2_WRAPFREE=$w python tools/prof_decoder.py --batch 65536 --reps 3 --precision fp16x2 --early-stop; done
