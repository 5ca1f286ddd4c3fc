# compute-sanitizer memcheck / racecheck / synccheck on a small wavefront + megakernel render
# (C1-sized Cornell box, light hierarchy, LPE layers), summaries into gpurun_out/sanitize_*.txt
cat > /tmp/san.py <<'PY'
import sys; sys.path.insert(0, ".")
from paper_1705_01263_b200 import scenes
from paper_1705_01263_b200.render import Renderer
from paper_1705_01263_b200.scene import pack_scene
import torch
for engine in ("wavefront", "megakernel"):
    # Cornell and 300 emitters: shared-memory BVHs; the 4096-triangle soup: global-memory BVH
    # (persistent lane-refill kernels on both placements); with and without LPE layers, FP64 and
    # compact path state, the three estimators
    for packed in (pack_scene(scenes.cornell()), pack_scene(scenes.many_lights(300), lights="tree"),
                   pack_scene(scenes.soup(4096)), pack_scene(scenes.envmap_scene(128, 64, sphere_subdiv=1))):
        for lpe, compact, est in ((True, False, "mis"), (False, False, "mis"), (False, True, "mis"),
                                  (False, False, "nee"), (False, True, "bsdf")):
            with Renderer(None, 24, 16, 5, packed=packed, engine=engine, pool_log2=10, compact_state=compact,
                          estimator=est) as r:
                if lpe:
                    r.set_lpe_layers({"d": "CD.*[LE]", "all": "C.*[LE]"})
                r.render_pass(0, 2)
                assert r.framebuffer().sum() > 0
                glob = torch.zeros((24 * 16, 3), dtype=torch.int64, device="cuda")
                r.set_stream(torch.cuda.current_stream().cuda_stream)
                r.accumulate_into(glob.data_ptr())
                torch.cuda.synchronize()
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
# the known-answer debug entries (BSDF, MIS, NEE light sampling, emission pdf) and the drop-in accel
timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_known_answers.py tests/test_gpu_accel.py \
  -m gpu -q -x -k "not bruteforce and not estimators_agree and not pdf_integral" > gpurun_out/sanitize_memcheck_known.txt 2>&1
echo "memcheck known-answer rc=$?" >> gpurun_out/sanitize_memcheck_known.txt
for f in gpurun_out/sanitize_memcheck_kernels.txt gpurun_out/sanitize_memcheck_bvh.txt; do tail -n 4 $f; done
