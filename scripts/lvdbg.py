import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1111_5572_b200 import api
tr = [("ACGTACGTAC" * 5, "ACGTACGTAC" * 5 + "GGGG", 16), ("ACGT" * 30, "ACGA" * 30, 40), ("A" * 200, "C" * 300, 20)]
print(api.bounded_distance_batch(tr), flush=True)
