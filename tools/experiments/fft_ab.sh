for r in 1 2; do for v in A B C D; do echo -n "$v "; python tools/prof_spectral.py --reps 3 --lib paper_2106_13062_b200/_lib/ab_$v.so; done; done
