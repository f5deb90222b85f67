"""One decode_sdr (or decode_hdr with --hdr) of a config-1 image, for profiling the serial decoder."""
import sys
sys.path.insert(0, ".")
import bench
import paper_2309_11072_b200 as P

pix = bench.generate(1, [0])[0]
h, w = pix.shape[:2]
st = P.encode(P.RadianceImage(w, h, pix, []))
(P.decode_hdr if "--hdr" in sys.argv else P.decode_sdr)(st)
