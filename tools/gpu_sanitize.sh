# compute-sanitizer memcheck / racecheck / synccheck on a small wavefront + megakernel render
# (C1-sized Cornell box, light hierarchy, LPE layers), summaries into gpurun_out/sanitize_*.txt
cat > /tmp/san.py <<'PY'
import sys; sys.path.insert(0, ".")
from paper_1705_01263_b200 import scenes
from paper_1705_01263_b200.render import Renderer
from paper_1705_01263_b200.scene import pack_scene
for engine in ("wavefront", "megakernel"):
    # Cornell and 300 emitters: shared-memory BVHs; the 4096-triangle soup: global-memory BVH
    # (persistent lane-refill kernels on both placements)
    for packed in (pack_scene(scenes.cornell()), pack_scene(scenes.many_lights(300), lights="tree"),
                   pack_scene(scenes.soup(4096))):
        with Renderer(None, 24, 16, 5, packed=packed, engine=engine, pool_log2=10) as r:
            r.set_lpe_layers({"d": "CD.*[LE]", "all": "C.*[LE]"})
            r.render_pass(0, 2)
            assert r.framebuffer().sum() > 0
print("ok")
PY
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.txt
done
for f in gpurun_out/sanitize_*.txt; do tail -n 3 $f; done
# the stateless kernel entry points and the BVH builders through their GPU tests
timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x \
  -k "not at_scale" > gpurun_out/sanitize_memcheck_kernels.txt 2>&1
echo "memcheck kernels rc=$?" >> gpurun_out/sanitize_memcheck_kernels.txt
timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_render.py -m gpu -q -x \
  -k "sah_tree_traversal or deep_sah or bvh_matches or warp_sah_decide and not soup1M" > gpurun_out/sanitize_memcheck_bvh.txt 2>&1
echo "memcheck bvh rc=$?" >> gpurun_out/sanitize_memcheck_bvh.txt
for f in gpurun_out/sanitize_memcheck_kernels.txt gpurun_out/sanitize_memcheck_bvh.txt; do tail -n 4 $f; done
