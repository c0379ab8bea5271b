"""Throughput of the C++ GA3C engine (ga3c_pipeline_run) on DNN A with
synthetic frame environments, over a grid of knobs (diagnostic, not the
bench).  usage: python tools/loop_probe.py [seconds]"""
import sys
import time

sys.path.insert(0, '.')
from paper_1611_06256_b200 import qac  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 5.0
grid = [  # (agents, predictors, trainers, pred_batch_max, device_frames)
    (128, 2, 2, 128, False),
    (128, 2, 2, 128, True),
    (128, 2, 3, 128, True),
    (128, 3, 3, 128, True),
    (256, 2, 3, 128, True),
    (256, 3, 4, 256, True),
]
for (na, npred, nt, pbm, dev) in grid:
    opt = qac.PipelineOptions(net=qac.dnn_a(), env=qac.frames(step_delay_us=0, episode_len=64), device_frames=dev)
    opt.knobs = qac.KnobConfig(n_agents=na, n_predictors=npred, n_trainers=nt, pred_batch_max=pbm, min_train_batch=40)
    opt.limits = (max(64, na), 16, 16)
    opt.stop = qac.StopCondition(max_seconds=secs)
    t0 = time.time()
    r = qac.run(opt)
    print(f"agents {na} pred {npred} train {nt} pbm {pbm} dev_frames {int(dev)}: samples/s {r.avg_samples_per_s:.0f} "
          f"pps {r.avg_pps:.0f} updates/s {r.avg_tps:.0f} batch {r.pred_batch_mean:.1f} lag {r.mean_lag:.1f} "
          f"wall {r.wall_time_s:.2f}", flush=True)
