// gen_trainer_golden.cpp — TEST INFRASTRUCTURE ONLY.  Runs the unmodified
// reference (proj/src/{trainer,model,dataset,layers,gns,tensor}.cpp, compiled
// in place from /root/reference by oracle/Makefile) and prints golden vectors
// for the GPU trainer (paper_2411_00999_b200/trainer.py):
//   * MarkovDataset streams (dataset.cpp:19-80): transition matrix and the
//     first sequences for a few (vocab, seed);
//   * make_toy_model weights (model.cpp:30-55) for one small config;
//   * scheduled_batch (trainer.cpp:25-32) at a grid of token counts;
//   * Trainer::step logs (trainer.cpp:284-426) of PerExample runs with SGD and
//     Adam, constant and cosine learning rate, fixed and ramped batch.
// Output: JSON on stdout (tests/golden/trainer_cases.json).
#include <cstdio>
#include <string>
#include <vector>

#include "gnstk/dataset.hpp"
#include "gnstk/model.hpp"
#include "gnstk/trainer.hpp"

using namespace gnstk;

static void arr(const std::vector<double>& v) {
    std::printf("[");
    for (size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? ", " : "", v[i]);
    std::printf("]");
}
static void arri(const std::vector<long long>& v) {
    std::printf("[");
    for (size_t i = 0; i < v.size(); ++i) std::printf("%s%lld", i ? ", " : "", v[i]);
    std::printf("]");
}
static void tensor(const Tensor& t) {
    std::vector<double> v(t.data(), t.data() + t.size());
    arr(v);
}

static void group(const char* name, const GroupLog& g) {
    std::printf("\"%s\": {\"g2_raw\": %.17g, \"s_raw\": %.17g, \"gns_ema\": %.17g, \"gns_defined\": %s}", name,
                g.g2_raw, g.s_raw, g.gns_ema, g.gns_defined ? "true" : "false");
}

static void run(const char* label, const TrainConfig& cfg, int steps, bool& first) {
    Trainer tr(cfg);
    std::printf("%s\n{\"family\": \"trainer\", \"label\": \"%s\", \"config\": {\"vocab\": %lld, \"model_dim\": %lld, "
                "\"hidden_multiplier\": %lld, \"n_blocks\": %lld, \"seq_len\": %lld, \"total_tokens\": %lld, "
                "\"optimizer\": \"%s\", \"beta1\": %.17g, \"beta2\": %.17g, \"eps\": %.17g, \"learning_rate\": %.17g, "
                "\"lr_schedule\": \"%s\", \"min_ratio\": %.17g, \"schedule\": \"%s\", \"b\": %lld, \"b_start\": %lld, "
                "\"b_end\": %lld, \"ramp_tokens\": %lld, \"ema_alpha\": %.17g, \"seed\": %llu, \"loss_scale\": %.17g}, "
                "\"steps\": [",
                first ? "" : ",", label, (long long)cfg.vocab, (long long)cfg.model_dim,
                (long long)cfg.hidden_multiplier, (long long)cfg.n_blocks, (long long)cfg.seq_len,
                (long long)cfg.total_tokens, cfg.optimizer.kind == OptimizerKind::Sgd ? "sgd" : "adam",
                cfg.optimizer.beta1, cfg.optimizer.beta2, cfg.optimizer.eps, cfg.learning_rate,
                cfg.lr_schedule.kind == LrScheduleKind::Constant ? "constant" : "cosine", cfg.lr_schedule.min_ratio,
                cfg.batch_schedule.kind == ScheduleKind::Fixed ? "fixed" : "linear_ramp", (long long)cfg.batch_schedule.b,
                (long long)cfg.batch_schedule.b_start, (long long)cfg.batch_schedule.b_end,
                (long long)cfg.batch_schedule.ramp_tokens, cfg.ema_alpha, (unsigned long long)cfg.seed, cfg.loss_scale);
    first = false;
    for (int s = 0; s < steps; ++s) {
        const StepLog log = tr.step();
        std::printf("%s\n {\"step\": %lld, \"tokens\": %lld, \"batch_size\": %lld, \"loss\": %.17g, ", s ? "," : "",
                    (long long)log.step, (long long)log.tokens, (long long)log.batch_size, log.loss);
        group("total", log.total);
        std::printf(", ");
        group("embedding", log.embedding);
        std::printf(", ");
        group("linear", log.linear);
        std::printf(", ");
        group("layernorm", log.layernorm);
        std::printf(", \"layers\": [");
        for (size_t i = 0; i < log.layers.size(); ++i)
            std::printf("%s{\"name\": \"%s\", \"g2_raw\": %.17g, \"s_raw\": %.17g}", i ? ", " : "",
                        log.layers[i].name.c_str(), log.layers[i].g2_raw, log.layers[i].s_raw);
        std::printf("]}");
    }
    std::printf("]}");
}

int main() {
    bool first = true;
    std::printf("[");
    // MarkovDataset streams
    for (auto [vocab, seed] : std::vector<std::pair<long long, unsigned long long>>{{2, 1}, {16, 1}, {16, 7}, {50, 123}}) {
        MarkovDataset d(vocab, seed);
        std::vector<long long> seqs;
        std::vector<std::int32_t> seq(17);
        for (int k = 0; k < 5; ++k) {
            d.fill_sequence(seq);
            for (auto v : seq) seqs.push_back(v);
        }
        std::printf("%s\n{\"family\": \"markov\", \"vocab\": %lld, \"seed\": %llu, \"transition\": ", first ? "" : ",",
                    vocab, seed);
        first = false;
        tensor(d.transition());
        std::printf(", \"seq_len\": 17, \"sequences\": ");
        arri(seqs);
        std::printf(", \"entropy_rate\": %.17g}", d.entropy_rate());
    }
    // make_toy_model weights
    {
        ToyModel m = make_toy_model(11, 6, 2, 2, 5);
        std::printf(",\n{\"family\": \"toy_init\", \"vocab\": 11, \"model_dim\": 6, \"hidden_multiplier\": 2, "
                    "\"n_blocks\": 2, \"seed\": 5, \"embed\": ");
        tensor(m.embed.weight);
        for (size_t i = 0; i < m.blocks.size(); ++i) {
            std::printf(", \"fc1_%zu\": ", i);
            tensor(m.blocks[i].fc1.weight);
            std::printf(", \"fc2_%zu\": ", i);
            tensor(m.blocks[i].fc2.weight);
        }
        std::printf(", \"head\": ");
        tensor(m.head.weight);
        std::printf("}");
    }
    // scheduled_batch
    {
        std::vector<long long> toks = {0, 1, 99, 100, 250, 499, 500, 501, 749, 750, 999, 1000, 5000};
        ScheduleSpec ramp{ScheduleKind::LinearRamp, 1, 3, 10, 1000};
        ScheduleSpec down{ScheduleKind::LinearRamp, 1, 4, 1, 600};
        ScheduleSpec fixed{ScheduleKind::Fixed, 32, 1, 1, 1};
        std::vector<long long> r, d2, f;
        for (auto t : toks) {
            r.push_back(scheduled_batch(ramp, t));
            d2.push_back(scheduled_batch(down, t));
            f.push_back(scheduled_batch(fixed, t));
        }
        std::printf(",\n{\"family\": \"schedule\", \"tokens\": ");
        arri(toks);
        std::printf(", \"ramp_3_10_1000\": ");
        arri(r);
        std::printf(", \"down_4_1_600\": ");
        arri(d2);
        std::printf(", \"fixed_32\": ");
        arri(f);
        std::printf("}");
    }
    // Trainer runs (PerExample)
    auto base = [] {
        TrainConfig c;
        c.vocab = 16;
        c.model_dim = 8;
        c.hidden_multiplier = 2;
        c.n_blocks = 2;
        c.seq_len = 8;
        c.total_tokens = 4096;
        c.learning_rate = 3e-3;
        c.ema_alpha = 0.2;
        c.seed = 3;
        c.batch_schedule = ScheduleSpec{ScheduleKind::Fixed, 6, 1, 1, 1};
        c.estimation_mode = EstimationMode{EstimationKind::PerExample, 1, 1};
        return c;
    };
    {
        TrainConfig c = base();
        c.optimizer.kind = OptimizerKind::Sgd;
        c.learning_rate = 0.1;
        run("sgd_fixed", c, 6, first);
    }
    {
        TrainConfig c = base();
        c.optimizer.kind = OptimizerKind::Adam;
        c.lr_schedule.kind = LrScheduleKind::Cosine;
        c.lr_schedule.min_ratio = 0.2;
        c.total_tokens = 400;
        c.batch_schedule = ScheduleSpec{ScheduleKind::LinearRamp, 1, 2, 7, 300};
        run("adam_cosine_ramp", c, 6, first);
    }
    {
        TrainConfig c = base();
        c.optimizer.kind = OptimizerKind::Sgd;
        c.learning_rate = 0.05;
        c.loss_scale = 2.5;
        c.vocab = 7;
        c.model_dim = 5;
        c.n_blocks = 1;
        c.seq_len = 5;
        c.seed = 11;
        run("sgd_loss_scale_odd_dims", c, 4, first);
    }
    std::printf("\n]\n");
    return 0;
}
