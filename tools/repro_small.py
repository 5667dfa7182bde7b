import sys
sys.path[:0] = ['tests', 'oracle', '.']
from helpers import load_corpus, groups, sub_batch
from paper_2405_07140_b200 import search
d = load_corpus('random_2024')
for algo in (1, 2):
    for lad, ids in list(groups(d).items())[:3]:
        b = sub_batch(d, ids)
        r = search.solve_batch(b, ladder=lad, algorithm=algo)
        print(algo, lad, r.z_found[:10])
