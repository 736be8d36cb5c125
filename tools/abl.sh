for es in "" "--early-stop"; do LSB_H2_WRAPFREE=1 python tools/prof_decoder.py --batch 65536 --reps 3 --precision fp16x2 $es; done
