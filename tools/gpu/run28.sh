timeout 300 python tools/step_profile.py alexconv_b128.opt.k0 30
timeout 300 python tools/step_profile.py vggconv_b64.opt.k0 12
