"""Throughput of the C++ GA3C engine (ga3c_pipeline_run) on DNN A with
synthetic frame environments, over a grid of knobs (diagnostic, not the
bench).  usage: python tools/loop_probe.py [seconds]"""
import os
import sys
import time

sys.path.insert(0, '.')
from paper_1611_06256_b200 import qac  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 5.0
grid = [  # (agents, predictors, trainers, pred_batch_max, device_frames, trainer_sms, predictor_sms)
    (256, 4, 6, 128, True, -1, -1),
    (256, 4, 8, 128, True, -1, -1),
    (384, 4, 6, 128, True, -1, -1),
    (384, 6, 8, 128, True, -1, -1),
    (256, 4, 6, 128, True, 0, 0),
    (512, 6, 8, 128, True, -1, -1),
]
for (na, npred, nt, pbm, dev, tsm, psm) in grid:
    opt = qac.PipelineOptions(net=qac.dnn_a(), env=qac.frames(step_delay_us=0, episode_len=64), device_frames=dev,
                              trainer_sms=tsm, predictor_sms=psm)
    opt.knobs = qac.KnobConfig(n_agents=na, n_predictors=npred, n_trainers=nt, pred_batch_max=pbm, min_train_batch=40)
    opt.limits = (max(64, na), 16, 16)
    opt.stop = qac.StopCondition(max_seconds=secs)
    t0 = time.time()
    c0 = os.times()
    r = qac.run(opt)
    c1 = os.times()
    cpu = (c1.user - c0.user + c1.system - c0.system) / (time.time() - t0)
    print(f"agents {na} pred {npred} train {nt} pbm {pbm} dev_frames {int(dev)} sms {tsm}/{psm}: samples/s {r.avg_samples_per_s:.0f} "
          f"pps {r.avg_pps:.0f} updates/s {r.avg_tps:.0f} batch {r.pred_batch_mean:.1f} lag {r.mean_lag:.1f} "
          f"wall {r.wall_time_s:.2f} cpu_cores_busy {cpu:.1f} (user {c1.user - c0.user:.1f}s sys {c1.system - c0.system:.1f}s)",
          flush=True)
