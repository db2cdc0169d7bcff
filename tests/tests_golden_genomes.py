"""Genome strings used by tests/golden/make_golden.py (kept in sync)."""
from paper_1909_12291_b200.genes import FIXED, SWEET, VGG16STYLE

SMALL = ("id=small00000000000 parents= lr=0.003 momentum=0.9 batch_size=8 "
         "f0=conv:oc=8,k=3,s=1,relu=1 f1=pool:size=2,s=2 f2=conv:oc=16,k=3,s=2,relu=1 h0=dense:units=12")
GENOMES = {"fixed": FIXED, "vgg16style": VGG16STYLE, "sweet": SWEET, "small": SMALL}
